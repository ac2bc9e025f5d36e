"""Summarise ncu output into profiles/ (run here, on the CPU box).

    python tools/ncu_summary.py --rep gpurun_out/prof_c2.ncu-rep --launches gpurun_out/launches_c2.csv \
        --workload c2_llama2_7b --algo-bytes 4296081664 --tag r01_c2

Writes profiles/<tag>_ncu.md (key metrics of the captured kernel, paper
Table 1/3 rows mapped to gb100 metrics as in SURVEY Appendix B), the launch
list of the step with each kernel's share, and merges the dominant kernel's
DRAM bytes per launch into profiles/ncu_summary.json (read by bench.py).
"""
import argparse
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

METRICS = [
    ("gpu__time_duration.sum", "Duration (paper Table 3 row 1)"),
    ("dram__bytes_read.sum", "DRAM bytes read"),
    ("dram__bytes_write.sum", "DRAM bytes written"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "Memory Throughput % (Table 3 row 3)"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "Compute Throughput % (Table 3 row 2)"),
    ("lts__t_sector_op_read_hit_rate.pct", "L2 read hit rate % (Table 3 row 4; includes prefetch-warmed lookups)"),
    ("lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum", "L2 tex read lookup hits (sectors)"),
    ("lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum", "L2 tex read lookup misses (sectors)"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit rate %"),
    ("smsp__average_warp_latency_per_inst_issued.ratio", "CPI-like: warp latency per issued inst (Table 3 row 5)"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "Stall Long Scoreboard (Table 3 row 6)"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "Stall barrier"),
    ("smsp__average_warps_issue_stalled_membar_per_issue_active.ratio", "Stall membar"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "Stall short scoreboard"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "Stall wait"),
    ("smsp__average_warps_issue_stalled_sleeping_per_issue_active.ratio", "Stall sleeping (mbarrier try_wait)"),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "Stall math pipe throttle"),
    ("l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum", "TMA load bytes"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "Tensor pipe active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "Achieved occupancy %"),
    ("launch__registers_per_thread", "Registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "Dynamic smem/block"),
    ("launch__occupancy_limit_shared_mem", "Occupancy limit (smem), CTAs/SM"),
    ("launch__grid_size", "Grid size"),
    ("launch__block_size", "Block size"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    kernels = []
    for vals in rows[2:]:
        kernels.append({h: (v, u) for h, v, u in zip(hdr, vals, units)})
    return kernels


def to_bytes(v, u):
    v = float(str(v).replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)
    return v * scale


def launches(path):
    lines = [l for l in open(path) if not l.startswith("==")]
    rows = list(csv.DictReader(lines))
    total = sum(float(r["Metric Value"]) for r in rows)
    return rows, total


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--workload", required=True)
    ap.add_argument("--algo-bytes", type=float, required=True)
    ap.add_argument("--tag", required=True)
    ap.add_argument("--kernel-filter", default="pda::")
    a = ap.parse_args()

    ks = raw(a.rep)
    md = [f"# ncu summary `{a.tag}` ({a.workload})", "",
          f"Source: `{os.path.basename(a.rep)}` (`ncu --set full --clock-control none --import-source on`, "
          "one B200, cold-cache serialised replay).", ""]
    summary = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json"))) \
        if os.path.exists(os.path.join(ROOT, "profiles", "ncu_summary.json")) else {}
    for k in ks:
        name = k.get("Kernel Name", ("?", ""))[0]
        md += [f"## `{name[:160]}`", "", "| metric | value | unit | meaning |", "|---|---|---|---|"]
        for m, meaning in METRICS:
            if m in k:
                v, u = k[m]
                md.append(f"| `{m}` | {v} | {u} | {meaning} |")
        rd = to_bytes(*k["dram__bytes_read.sum"]) if "dram__bytes_read.sum" in k else None
        wr = to_bytes(*k["dram__bytes_write.sum"]) if "dram__bytes_write.sum" in k else 0
        if rd is not None:
            traffic = rd + wr
            md += ["", f"DRAM traffic per launch = {traffic:.4e} B; algorithmic bytes = {a.algo_bytes:.4e} B; "
                   f"ratio = {traffic / a.algo_bytes:.4f}", ""]
            if "splitk_kernel" in name or "balanced_kernel" in name:
                summary[a.workload] = {"dram_bytes_per_launch": traffic, "kernel": name[:120],
                                       "algorithmic_bytes": a.algo_bytes, "tag": a.tag}
    if a.launches:
        rows, total = launches(a.launches)
        md += ["## Launch list of the step (`--metrics gpu__time_duration.sum`)", "",
               "| # | kernel | grid | block | ns | share of all launches | share of step (pda kernels) |",
               "|---|---|---|---|---|---|---|"]
        ours = [r for r in rows if a.kernel_filter in r["Kernel Name"]]
        ours_total = sum(float(r["Metric Value"]) for r in ours) or 1.0
        for r in rows:
            v = float(r["Metric Value"])
            mine = a.kernel_filter in r["Kernel Name"]
            md.append(f"| {r['ID']} | `{r['Kernel Name'].split('(')[0][:70]}` | {r['Grid Size']} | {r['Block Size']} | "
                      f"{v:.0f} | {v / total:.3f} | {(v / ours_total) if mine else 0:.3f} |")
        md.append("")
        md.append("Setup launches (torch RNG / fills) precede the timed steps; the step itself is the pda kernels.")
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"{a.tag}_ncu.md"), "w") as f:
        f.write("\n".join(md) + "\n")
    with open(os.path.join(ROOT, "profiles", "ncu_summary.json"), "w") as f:
        json.dump(summary, f, indent=1)
    print("\n".join(md[:60]))


if __name__ == "__main__":
    main()
