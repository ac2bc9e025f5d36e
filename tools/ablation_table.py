"""Turn ncu ablation CSVs (tools/ablation_launches.py under `ncu --metrics`)
into the paper-Table-3-style markdown table in profiles/.

    python tools/ablation_table.py gpurun_out/ablation_c2.csv ... > profiles/r01_prefetch_ablation_ncu.md
"""
import csv
import json
import os
import sys
from collections import OrderedDict

ROWS = [
    ("gpu__time_duration.sum", "Duration (us)", 1e-3),
    ("dram__bytes_read.sum", "DRAM read (MB)", None),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "Memory Throughput (%)", 1),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM Throughput (%)", 1),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "Compute Throughput (%)", 1),
    ("lts__t_sector_op_read_hit_rate.pct", "L2 read hit rate (%)", 1),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit rate (%)", 1),
    ("smsp__average_warp_latency_per_inst_issued.ratio", "Cycles per issued inst (CPI)", 1),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "Stall Long Scoreboard (cycles)", 1),
    ("smsp__average_warps_issue_stalled_sleeping_per_issue_active.ratio", "Stall sleeping (mbarrier wait)", 1),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "Stall wait", 1),
    ("smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio", "Stall LG throttle", 1),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "Achieved occupancy (%)", 1),
]


def label(v):
    s = v["kernel"]
    if v["kernel"] == "splitk":
        s += f" S{v['smem_stages']}" if v.get("smem_stages") else " default ring"
        if v.get("issue_mode"):
            s += f" {v['issue_mode']}"
        if v.get("kv"):
            s += f" {v['kv']}"
    s += " " + v["prefetch"]
    if v["prefetch"] != "off":
        s += f" d{v['prefetch_distance']}"
    if v.get("eviction"):
        s += f" {v['eviction']}"
    return s


def load(path):
    lines = [l for l in open(path) if not l.startswith("==")]
    rows = list(csv.DictReader(lines))
    kern = OrderedDict()
    for r in rows:
        kern.setdefault(r["ID"], {})[r["Metric Name"]] = (r["Metric Value"], r["Metric Unit"])
    order = json.load(open(path.replace("ablation_", "ablation_order_").replace(".csv", ".json")))
    out = []
    for (kid, m), v in zip(kern.items(), order):
        if v["rep"] == 1:
            out.append((label(v), m, v))
    return out


def fmt(m, key, scale):
    if key not in m:
        return "-"
    val, unit = m[key]
    x = float(val.replace(",", ""))
    if key == "gpu__time_duration.sum":
        x = x * {"ns": 1e-3, "us": 1, "ms": 1e3}.get(unit, 1)
        return f"{x:.1f}"
    if key == "dram__bytes_read.sum":
        x = x * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1, "Gbyte": 1e3}.get(unit, 1)
        return f"{x:.0f}"
    return f"{x:.2f}"


def summary(paths):
    """One row per cell: duration, L2 read hit rate and long-scoreboard share
    of CPI with prefetch off / on, and the speedup, for every variant."""
    hdr = None
    for path in paths:
        cfg = os.path.basename(path)[len("ablation_"):-4]
        full = load(path)
        base = {}
        for c, m, v in full:
            if v["prefetch"] == "off":
                base[(v["kernel"], v.get("issue_mode"), v.get("kv"))] = m
        if hdr is None:
            hdr = [c for c, _, v in full if v["prefetch"] != "off"]
            print("| cell | " + " | ".join(f"{c}: speedup / L2 hit off->on / LS share off->on" for c in hdr) + " |")
            print("|---|" + "---|" * len(hdr))
        cells = []
        for c, m, v in full:
            if v["prefetch"] == "off":
                continue
            m0 = base[(v["kernel"], v.get("issue_mode"), v.get("kv"))]
            d0 = float(m0["gpu__time_duration.sum"][0])
            d1 = float(m["gpu__time_duration.sum"][0])
            h0 = float(m0["lts__t_sector_op_read_hit_rate.pct"][0])
            h1 = float(m["lts__t_sector_op_read_hit_rate.pct"][0])

            def ls(x):
                return 100 * float(x["smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio"][0]) / \
                    float(x["smsp__average_warp_latency_per_inst_issued.ratio"][0])
            cells.append(f"{d0 / d1:.3f}x / {h0:.0f}->{h1:.0f}% / {ls(m0):.0f}->{ls(m):.0f}%")
        print(f"| {cfg} | " + " | ".join(cells) + " |")


def main():
    if sys.argv[1] == "--summary":
        summary(sys.argv[2:])
        return
    for path in sys.argv[1:]:
        cfg = os.path.basename(path)[len("ablation_"):-4]
        full = load(path)
        cols = [(c, m) for c, m, _ in full]
        print(f"### {cfg}\n")
        print("| metric | " + " | ".join(c for c, _ in cols) + " |")
        print("|---|" + "---|" * len(cols))
        for key, name, scale in ROWS:
            print(f"| {name} | " + " | ".join(fmt(m, key, scale) for _, m in cols) + " |")
        # long-scoreboard share of CPI, as the paper quotes (21.34 / 27.68 = 77%)
        shares = []
        for _, m in cols:
            try:
                ls = float(m["smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio"][0])
                cpi = float(m["smsp__average_warp_latency_per_inst_issued.ratio"][0])
                shares.append(f"{100 * ls / cpi:.0f}%")
            except Exception:
                shares.append("-")
        print("| Long-scoreboard share of CPI | " + " | ".join(shares) + " |")
        d0 = [float(m["gpu__time_duration.sum"][0]) for _, m in cols]
        base = {}
        sp = []
        for (c, m, v), d in zip(full, d0):
            fam = (v["kernel"], v.get("issue_mode"), v.get("kv"))  # same kernel, any ring depth
            if v["prefetch"] == "off":
                base[fam] = d
            sp.append(f"{base.get(fam, d) / d:.3f}x")
        print("| Speedup vs same kernel, prefetch off | " + " | ".join(sp) + " |\n")


if __name__ == "__main__":
    main()
