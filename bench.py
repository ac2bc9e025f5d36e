"""Benchmark: B200 paged decode attention with L2 KV prefetch (arXiv 2504.06319).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

One "step" is one decode-attention pass over the whole batch (every row of
the hot-path table: plan, block-table walk, L2 prefetch, KV load, QK^T,
online softmax, PV, combine; plus the TP output all-gather when N > 1).
Inputs are seeded synthetic tensors shaped like BASELINE.json's configs
(default configs[1], Llama-2-7B: B=64, 32 heads, D=128, ctx 4096, fp16),
resident in HBM before the timed region; KV per step (4.3 GB) is far larger
than L2 (126 MB), so no flush is needed between steps (smaller --config
cells, KV < 4 x L2, flush L2 between individually timed steps).

N > 1 (torchrun): tensor parallel over KV heads -- rank r holds
Hkv/N heads of the same batch and the step ends with an NCCL all-gather of
the output heads; the total work is fixed (strong scaling).

Prints ONE JSON line (rank 0).  `value` = algorithmic KV+q+out bytes moved
per step, all ranks, / max-over-ranks device time (GB/s).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode attention us/step & achieved HBM GB/s (prefetch on/off); tokens/s at 1-8 GPU"
KERNEL_NAMES = {1: "paper_kernel", 2: "splitk_kernel", 3: "stream_kernel", 4: "balanced_kernel", 5: "tc_kernel"}


L2_BYTES = 126 * 1024 * 1024  # B200 L2


class L2Flush:
    """Evict L2 between timed steps without leaving it dirty: write 512 MiB
    (every line of the previous step evicted), then read 256 MiB of another
    buffer, so the lines the write left dirty are written back here, outside
    the timed span, and not by the next step's loads (a write-only flush
    charged the next step up to 126 MB of write-back, ~17 us)."""

    def __init__(self, torch):
        self.w = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
        self.r = torch.ones(128 << 20, dtype=torch.float16, device="cuda")
        self.sink = torch.empty((), dtype=torch.float32, device="cuda")
        self.torch = torch

    def __call__(self):
        self.w.zero_()
        self.torch.sum(self.r, dim=0, dtype=self.torch.float32, out=self.sink)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--prefetch", default=None, help="bulk|line|off (default: library default)")
    ap.add_argument("--distance", type=int, default=None)
    ap.add_argument("--stages", type=int, default=0)
    ap.add_argument("--partition", type=int, default=0)
    ap.add_argument("--kernel", default=None, help="auto|splitk|balanced|stream|paper|tc")
    ap.add_argument("--no-extras", action="store_true", help="skip ablation arms / e2e / cpu baseline")
    ap.add_argument("--fused-gather", action="store_true",
                    help="TP output all-gather inside the kernel's stores (symmetric memory) instead of NCCL")
    ap.add_argument("--nccl-gather", action="store_true",
                    help="N > 1: always gather with NCCL (default: the fused gather when its first step "
                         "matches the NCCL step bitwise on every rank)")
    ap.add_argument("--sweep", action="store_true", help="prefetch-distance x stages sweep (extra JSON lines on stderr)")
    return ap.parse_args()


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def load_traffic(workload: str):
    """dram bytes per launch of the dominant kernel from the committed ncu summary."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get(workload, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            parts = [p.strip() for p in l.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        loaded = [s for s in sm if s > 0.5 * (mx or max(sm))] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def workload_config(name: str):
    import synth
    if name in synth.PRESETS:
        return synth.PRESETS[name]
    if name.startswith("c4_"):  # c4_b{B}_ctx{C}
        _, b, c = name.split("_")
        return synth.sweep_cell(int(b[1:]), int(c[3:]))
    if name.startswith("u_"):  # u_B_Hq_Hkv_D_ctx_dtype: a uniform custom shape
        _, B, Hq, Hkv, D, ctx, dt = name.split("_")
        return synth.uniform(name, int(B), int(Hq), int(Hkv), int(D), int(ctx), dt)
    raise SystemExit(f"unknown config {name}")


def algorithmic_bytes(cfg, out_elem=2):
    """KV + q + out + block-table + lens bytes one step must move."""
    return cfg.kv_bytes() + cfg.other_bytes(out_elem)


def spread(xs):
    """median, p10, p90 (nearest-rank on the sorted sample) and n of a list of times."""
    xs = sorted(xs)
    n = len(xs)

    def q(f):
        return xs[min(n - 1, max(0, int(round(f * (n - 1)))))]
    return {"median": statistics.median(xs), "p10": q(0.10), "p90": q(0.90), "n": n}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


# ------------------------------------------------------------------ CPU oracle legs
def oracle_sample(cfg, seconds: float, seed: int = 0):
    """Time the fp64 oracle (as it stands) on whole sequences of the workload
    until ~`seconds` of wall time; returns (GB/s, sample description, threads)."""
    import numpy as np
    import torch

    import oracle
    import synth
    oracle.build()
    threads = len(os.sched_getaffinity(0))
    one = synth.Config(cfg.name + "_sample", 1, cfg.num_q_heads, cfg.num_kv_heads, cfg.head_dim,
                       (cfg.context_lens[0],), cfg.dtype)
    inp = synth.make_inputs(one, seed=seed)
    nbytes = algorithmic_bytes(one)
    done, t0 = 0, time.perf_counter()
    while True:
        oracle.paged_attention(inp["q"], inp["k_cache"], inp["v_cache"], inp["block_tables"],
                               inp["context_lens"], inp["scale"], one.dtype, nthreads=threads)
        done += 1
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    gbs = done * nbytes / el / 1e9
    desc = (f"{done} x one sequence of {cfg.name} (all {cfg.num_q_heads} q heads, ctx "
            f"{cfg.context_lens[0]}), fp64 oracle, {el:.2f} s wall")
    return gbs, desc, threads, el / done


def run_reference(args, rank, world):
    """--impl reference: the oracle is this tier's reference arm (rank 0 only)."""
    if rank != 0:
        return
    cfg = workload_config(args.config)
    # per step: one sequence of the workload (bounded sample); value scaled as GB/s
    gbs_w, desc, threads, _ = oracle_sample(cfg, 0.5)
    times = []
    import oracle
    import synth
    one = synth.Config(cfg.name + "_sample", 1, cfg.num_q_heads, cfg.num_kv_heads, cfg.head_dim,
                       (cfg.context_lens[0],), cfg.dtype)
    inp = synth.make_inputs(one, seed=1)
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        oracle.paged_attention(inp["q"], inp["k_cache"], inp["v_cache"], inp["block_tables"],
                               inp["context_lens"], inp["scale"], one.dtype, nthreads=threads)
        if i >= args.warmup:
            times.append(time.perf_counter() - t0)
    per = sum(times) / len(times)
    value = algorithmic_bytes(one) / per / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": per * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": cfg.name, "sample": "one sequence per step (all heads)"},
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": threads, "kind": "oracle",
                         "sample": f"one sequence of {cfg.name} per step, {args.steps} steps",
                         "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU leg
def main():
    args = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    import paper_2504_06319_b200 as pda
    import synth
    from paper_2504_06319_b200.tp import TPDecodeAttention

    # PDA_BENCH_SHARE_GPU=1 (testing only): ranks share the visible GPUs round-robin
    # and use gloo, so the multi-rank path can be exercised on a 1-GPU box
    share = os.environ.get("PDA_BENCH_SHARE_GPU") == "1"
    dev_index = local % torch.cuda.device_count() if share else local
    torch.cuda.set_device(dev_index)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_index))
    # PDA_BENCH_CHECK_FUSED=1 (testing only): run the N > 1 fused-gather selection at N = 1
    check_fused_1 = os.environ.get("PDA_BENCH_CHECK_FUSED") == "1" and world == 1
    if world == 1 and (args.fused_gather or check_fused_1):  # symmetric memory needs a process group
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", dev_index))
    pda.lib()

    cfg = workload_config(args.config)
    if cfg.num_kv_heads % world:
        raise SystemExit(f"{cfg.num_kv_heads} KV heads do not shard over {world} GPUs")
    local_cfg = cfg.with_heads(cfg.num_q_heads // world, cfg.num_kv_heads // world,
                               name=f"{cfg.name}_tp{world}_rank{rank}")
    inp = synth.make_inputs(local_cfg, seed=1234 + rank, device="cuda", poison=True)
    dt = synth.torch_dtype(cfg.dtype)
    opt_kw = {}
    if args.prefetch is not None:
        opt_kw["prefetch"] = args.prefetch
    if args.distance is not None:
        opt_kw["prefetch_distance"] = args.distance
    if args.stages:
        opt_kw["smem_stages"] = args.stages
    if args.partition:
        opt_kw["partition_tokens"] = args.partition
    if args.kernel:
        opt_kw["kernel"] = args.kernel

    def make_step(**kw):
        return TPDecodeAttention(inp["k_cache"], inp["v_cache"], local_cfg.num_seqs,
                                 local_cfg.num_q_heads, local_cfg.max_blocks_per_seq, dt, **kw)

    step_main = make_step(**opt_kw, fused_gather=args.fused_gather)
    q, bt, lens, scale = inp["q"], inp["block_tables"], inp["context_lens"], inp["scale"]
    stream = torch.cuda.current_stream()
    tp_gather = "fused" if args.fused_gather else "nccl"
    step_nccl = None
    if (world > 1 or check_fused_1) and not share and not args.fused_gather and not args.nccl_gather:
        # fused output all-gather when it works here: its first
        # step must equal the NCCL step bit for bit on every rank, else NCCL
        def all_ok(ok):  # every rank agrees before anyone enters a cross-rank device barrier
            flag = torch.tensor([ok], dtype=torch.int32, device="cuda")
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)
            return int(flag.item()) == 1

        ok = 1
        try:
            step_fused = make_step(**opt_kw, fused_gather=True)
        except Exception as e:  # noqa: BLE001 -- any failure selects the NCCL path
            print(f"[bench rank {rank}] fused gather unavailable: {e}", file=sys.stderr)
            ok = 0
        if all_ok(ok):
            try:
                ref = step_main(q, bt, lens, scale).reshape(local_cfg.num_seqs, -1, cfg.head_dim).clone()
                got = step_fused(q, bt, lens, scale).reshape(local_cfg.num_seqs, -1, cfg.head_dim).clone()
                torch.cuda.synchronize()
                ok = int(torch.equal(ref.view(torch.int16), got.view(torch.int16)))
            except Exception as e:  # noqa: BLE001
                print(f"[bench rank {rank}] fused gather failed: {e}", file=sys.stderr)
                ok = 0
        else:
            ok = 0
        if all_ok(ok):
            step_nccl, step_main, tp_gather = step_main, step_fused, "fused"

    def barrier():
        if world > 1:
            dist.barrier()

    # steps whose KV fits in a few L2s would hit in L2 across back-to-back
    # steps: flush it between timed steps (outside the timed spans)
    flush_buf = L2Flush(torch) if local_cfg.kv_bytes() < 4 * L2_BYTES else None

    step_spread = {}

    def time_steps(fn, steps, warmup, join=None, key=None, join_end=None):
        """Mean device ms per step over `steps` timed steps (max over ranks); with
        `key`, the per-step spread (median / p10 / p90, us) is kept in step_spread.
        join: multi-stream steps, the timer's stream waits for all of them after
        every step; join_end: only once, after the last step (a pipelined loop:
        step k's side-stream copies overlap step k + 1's kernels; the span still
        ends after every copy of every step)."""
        for _ in range(warmup):
            fn(q, bt, lens, scale)
        if join:
            join(stream)
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        if flush_buf is not None:
            spans = []
            for _ in range(steps):
                flush_buf()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                fn(q, bt, lens, scale)
                if join or join_end:  # individually timed (flushed) steps: every step's copies inside
                    (join or join_end)(stream)
                e1.record(stream)
                spans.append((e0, e1))
            torch.cuda.synchronize()
            barrier()
            per = [a.elapsed_time(b) for a, b in spans]
            ms = sum(per) / steps
        else:
            # back-to-back steps, an event between consecutive steps: the K
            # intervals are the per-step times, their sum the span of the K steps
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
            ev[0].record(stream)
            for i in range(steps):
                fn(q, bt, lens, scale)
                if join:
                    join(stream)  # multi-stream steps: the timer's stream waits for all of them
                if join_end and i == steps - 1:
                    join_end(stream)
                ev[i + 1].record(stream)
            torch.cuda.synchronize()
            barrier()
            per = [ev[i].elapsed_time(ev[i + 1]) for i in range(steps)]
            ms = ev[0].elapsed_time(ev[-1]) / steps
        if world > 1:
            t = torch.tensor([ms], device="cpu" if share else "cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        if key is not None:
            step_spread[key] = {k: (v * 1e3 if k != "n" else v) for k, v in spread(per).items()}
        return ms

    total_bytes = algorithmic_bytes(cfg)  # whole job (all ranks' shards)
    local_bytes = algorithmic_bytes(local_cfg)
    peak, peak_src = load_peaks()

    with ClockSampler(dev_index) as clk:
        ms = time_steps(step_main, args.steps, args.warmup, key="step")
        extras = {}
        if step_nccl is not None:  # the NCCL-gather step, for comparison with the fused one
            extras["tp_nccl_gather_us_per_step"] = time_steps(step_nccl, args.steps, 2) * 1e3
        if not args.no_extras:
            # prefetch ablation arms on the same inputs, interleaved step by step
            # (A B A B ...) with per-step CUDA events, medians per arm
            arms = {
                "on": make_step(**{**opt_kw, "prefetch": "line", "prefetch_distance": 4}),
                "bulk": make_step(**{**opt_kw, "prefetch": "bulk", "prefetch_distance": 4}),
                "off": make_step(**{**opt_kw, "prefetch": "off"}),
                "paper_on": make_step(kernel="paper", prefetch="bulk", prefetch_distance=4),
                "paper_off": make_step(kernel="paper", prefetch="off"),
                # the paper kernel as prefetch AUTO runs it on short GQA steps: line d4, evict_last
                "paper_line_el": make_step(kernel="paper", prefetch="line", prefetch_distance=4,
                                           eviction="prefetch_last"),
            }
            tc_ok = cfg.head_dim == 128 and getattr(local_cfg, "kv_dtype", "") != "e4m3"
            if tc_ok:  # the tcgen05 kernel (decode_tc.cu) on the same step
                arms["tc"] = make_step(kernel="tc", prefetch="off")
            per = {k: [] for k in arms}
            for k, fn in arms.items():  # warm each arm
                fn(q, bt, lens, scale)
            torch.cuda.synchronize()
            n_rep = max(50, args.steps)
            for _ in range(n_rep):
                for k, fn in arms.items():
                    if flush_buf is not None:
                        flush_buf()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    fn(q, bt, lens, scale)
                    e1.record(stream)
                    per[k].append((e0, e1))
            torch.cuda.synchronize()
            us = {k: [a.elapsed_time(b) * 1e3 for a, b in v] for k, v in per.items()}
            med = {k: statistics.median(v) for k, v in us.items()}

            def ratio(off, on):  # paired per round (the arms of one round ran back to back)
                return spread([a / b for a, b in zip(us[off], us[on])])
            extras = {
                "prefetch_on_us": med["on"],
                "prefetch_off_us": med["off"],
                "prefetch_speedup": med["off"] / med["on"],
                "prefetch_on_desc": "same kernel + prefetch.global.L2 line prefetch 4 blocks ahead",
                "prefetch_bulk_us": med["bulk"],
                "prefetch_bulk_speedup": med["off"] / med["bulk"],
                "paper_kernel": {
                    "prefetch_on_us": med["paper_on"],
                    "prefetch_off_us": med["paper_off"],
                    "prefetch_speedup": med["paper_off"] / med["paper_on"],
                    "desc": "paper structure: grid [Hq,B], 4 warps, warp-per-block LDG, Alg. 1 bulk d=4",
                    "line_d4_evict_last_us": med["paper_line_el"],
                    "line_d4_evict_last_speedup": med["paper_off"] / med["paper_line_el"],
                },
                "arms_us": {k: spread(v) for k, v in us.items()},
                "speedup_spread": {"line_d4": ratio("off", "on"), "bulk_d4": ratio("off", "bulk"),
                                   "paper_bulk_d4": ratio("paper_off", "paper_on"),
                                   "paper_line_d4_evict_last": ratio("paper_off", "paper_line_el")},
                "arms_timing": f"{n_rep} interleaved rounds (A B C D E, A B C D E, ...), per-step CUDA events; "
                               f"medians, p10/p90; speedups = off/on paired per round",
            }
            if "tc" in med:
                extras["tc_kernel"] = {
                    "us_per_step": med["tc"], "speedup_vs_default": med["off"] / med["tc"],
                    "spread_us": spread(us["tc"]), "gbs": local_bytes / (med["tc"] * 1e3),
                    "desc": "tcgen05 kernel: persistent CTA per SM, QK^T / PV on tcgen05.mma with S, O in TMEM "
                            "(kernel='tc'; not the default: slower than split-K here)"}
            # FP8 (e4m3) KV-cache variant of the same step
            if cfg.head_dim == 128:
                q8 = synth.quantize_kv_e4m3(inp)
                ws8 = torch.zeros(max(1, pda.workspace_bytes(
                    pda.make_shape(q, q8["k_cache"], bt), pda.make_options(**opt_kw))), dtype=torch.uint8,
                    device="cuda")

                def kv8_step(q_, bt_, lens_, scale_):
                    pda.paged_decode_attention(q_, q8["k_cache"], q8["v_cache"], bt_, lens_, scale_,
                                               out=step_main.out_local, workspace=ws8, k_scale=q8["k_scale"],
                                               v_scale=q8["v_scale"], **opt_kw)
                ms8 = time_steps(kv8_step, max(10, args.steps // 2), 2)
                b8 = cfg.kv_bytes() // 2 + cfg.other_bytes()
                extras["e4m3_kv"] = {"us_per_step": ms8 * 1e3, "speedup_vs_16bit": ms / ms8,
                                     "algorithmic_gbs": b8 / (ms8 * 1e-3) / 1e9 * world,
                                     "tokens_per_s": cfg.num_seqs / (ms8 * 1e-3),
                                     "desc": "K/V as OCP e4m3 codes + per-tensor scales, 1 B/element"}
                del q8, ws8
            # the decode step with its KV append (SURVEY 8f NEXT f3 alternative):
            # fused into the split-K kernel vs a separate append launch first
            kn, vn = synth.new_kv_rows(inp, 1, seed=rank)

            def app_fused():
                pda.paged_decode_attention(q, inp["k_cache"], inp["v_cache"], bt, lens, scale,
                                           out=step_main.out_local, workspace=step_main.ws, k_new=kn, v_new=vn,
                                           **opt_kw)

            def app_separate():
                pda.kv_append(kn, vn, inp["k_cache"], inp["v_cache"], bt, lens)
                pda.paged_decode_attention(q, inp["k_cache"], inp["v_cache"], bt, lens, scale,
                                           out=step_main.out_local, workspace=step_main.ws, **opt_kw)

            def app_none():
                pda.paged_decode_attention(q, inp["k_cache"], inp["v_cache"], bt, lens, scale,
                                           out=step_main.out_local, workspace=step_main.ws, **opt_kw)

            app_arms = {"fused": app_fused, "separate": app_separate, "attention_only": app_none}
            app_per = {k: [] for k in app_arms}
            for fn in app_arms.values():
                fn()
            torch.cuda.synchronize()
            for _ in range(max(10, args.steps // 4)):
                for k, fn in app_arms.items():
                    if flush_buf is not None:
                        flush_buf()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    fn()
                    e1.record(stream)
                    app_per[k].append((e0, e1))
            torch.cuda.synchronize()
            am = {k: statistics.median(a.elapsed_time(b) for a, b in v) * 1e3 for k, v in app_per.items()}
            extras["kv_append"] = {
                "fused_us": am["fused"], "separate_us": am["separate"], "attention_only_us": am["attention_only"],
                "desc": "step = append the new token's K/V into its paged slot + attention; fused: the split-K "
                        "CTA owning the slot writes it before its TMA loads (one launch fewer)"}
            del kn, vn
            # in-run read roofline (read-only streams over a 4 GiB buffer): LDG.128 and
            # two bulk-copy (TMA engine) variants, the best of them is the ceiling
            buf = torch.empty(4 << 30, dtype=torch.uint8, device="cuda")
            sink = torch.zeros(4, dtype=torch.int32, device="cuda")
            probe = {}
            for mode in ("ldg", "bulk16k", "bulk_ring"):
                for _ in range(2):
                    pda.read_roofline(buf, sink, mode=mode)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                for _ in range(5):
                    pda.read_roofline(buf, sink, mode=mode)
                e1.record(stream)
                torch.cuda.synchronize()
                probe[mode] = buf.numel() * 5 / (e0.elapsed_time(e1) * 1e-3) / 1e9
            extras["read_roofline_probes_gbs"] = probe
            extras["read_roofline_gbs"] = max(probe.values())
            del buf
            # Eq. 1-2 and the L2 residency bound re-derived for this device (DESIGN 7.5)
            l2 = getattr(torch.cuda.get_device_properties(dev_index), "L2_cache_size", L2_BYTES)
            m_block = 16 * cfg.head_dim * 2  # Eq. 1: b * d_h * T_block
            m_total_b1 = m_block * (128 // 32) * cfg.num_q_heads  # Eq. 2 at B=1 (paper kernel, K blocks)
            plan = step_main.plan
            sms = torch.cuda.get_device_properties(dev_index).multi_processor_count
            resident = sms * (3 if plan["smem_stages"] >= 8 else 4)
            extras["l2_capacity"] = {
                "l2_bytes": l2, "m_block_bytes": m_block, "paper_kernel_m_total_b1_bytes": m_total_b1,
                "residency_bound_batches": l2 // m_total_b1,
                "splitk_prefetch_lookahead_bytes_per_block_of_distance": resident * 2 * m_block,
                "splitk_distance_filling_l2": l2 // (resident * 2 * m_block),
                "desc": "paper: 60 MB L2 / 512 KiB = 120 batches (P:180); split-K: resident CTAs x d x "
                        "(K+V) M_block of L2 lookahead beyond the smem ring"}

    # the dominant kernel's own launch time (attention call alone, no gather)
    def attn_only(q_, bt_, lens_, scale_):
        pda.paged_decode_attention(q_, inp["k_cache"], inp["v_cache"], bt_, lens_, scale_,
                                   out=step_main.out_local, workspace=step_main.ws, **opt_kw)
    attn_ms = time_steps(attn_only, args.steps, 2, key="attention")
    achieved = local_bytes / (attn_ms * 1e-3) / 1e9

    # the same attention call captured in a CUDA graph (a serving loop replays the
    # decode step this way; it removes the Python + C-ABI host cost per launch,
    # which dominates steps of a few tens of microseconds)
    graph = None
    if not args.no_extras:
        gr = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        side.wait_stream(stream)
        with torch.cuda.stream(side):
            attn_only(q, bt, lens, scale)
        stream.wait_stream(side)
        with torch.cuda.graph(gr):
            attn_only(q, bt, lens, scale)
        graph_ms = time_steps(lambda *_: gr.replay(), args.steps, 2, key="graph")
        graph = {"us_per_step": graph_ms * 1e3, "eager_us_per_step": attn_ms * 1e3,
                 "gbs": local_bytes / (graph_ms * 1e-3) / 1e9, "spread_us": step_spread["graph"],
                 "desc": "attention call (this rank) captured once in a CUDA graph and replayed; eager = the "
                         "same call launched from Python through the C ABI"}
        del gr

    # end to end through the public C-ABI host entry (pinned host q/bt/lens in, out back)
    e2e = None
    if not args.no_extras and world == 1:
        host = pda.HostDecodeStep(inp["k_cache"], inp["v_cache"], local_cfg.num_seqs,
                                  local_cfg.num_q_heads, local_cfg.max_blocks_per_seq, dt, slots=2, **opt_kw)
        qh, bth, lh = q.cpu().pin_memory(), bt.cpu().pin_memory(), lens.cpu().pin_memory()

        def e2e_step(*_):
            host(qh, bth, lh, scale)
        e2e_ms = time_steps(e2e_step, max(10, args.steps // 2), 2, join_end=host.join)
        e2e = {"value": total_bytes / (e2e_ms * 1e-3) / 1e9, "unit": "GB/s",
               "ms_per_step": e2e_ms, "h2d_bytes_per_step": host.h2d_bytes(),
               "d2h_bytes_per_step": host.d2h_bytes(),
               "path": "pda_decode_step_host (H2D q/bt/lens from pinned memory, kernels, D2H out), "
                       "2 staging slots, copies on per-slot copy streams overlapping the neighbouring steps' kernels; "
                       "kernels in order on one stream; the timed span ends after the last step's D2H"}
    elif not args.no_extras:
        # N > 1: the TP step end to end -- this rank's q slice, the tables and the
        # lengths from pinned host memory, the kernels, the output all-gather
        # (the step's collective), and the gathered [B, Hq, D] output back to the host
        qh, bth, lh = q.cpu().pin_memory(), bt.cpu().pin_memory(), lens.cpu().pin_memory()
        qd, btd, ld = torch.empty_like(q), torch.empty_like(bt), torch.empty_like(lens)
        out_h = torch.empty((cfg.num_seqs, cfg.num_q_heads, cfg.head_dim), dtype=dt).pin_memory()

        def e2e_step(*_):
            qd.copy_(qh, non_blocking=True)
            btd.copy_(bth, non_blocking=True)
            ld.copy_(lh, non_blocking=True)
            g = step_main(qd, btd, ld, scale)
            out_h.copy_(g.reshape(out_h.shape), non_blocking=True)
        e2e_ms = time_steps(e2e_step, max(10, args.steps // 2), 2)
        h2d = (qh.numel() * qh.element_size() + bth.numel() * 4 + lh.numel() * 4) * world
        e2e = {"value": total_bytes / (e2e_ms * 1e-3) / 1e9, "unit": "GB/s",
               "ms_per_step": e2e_ms, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": out_h.numel() * out_h.element_size() * world,
               "path": f"TPDecodeAttention per rank: H2D of the rank's q slice / tables / lengths from pinned "
                       f"memory, the kernels, the {tp_gather} output all-gather, D2H of the gathered output "
                       f"(every rank), one stream; max over ranks"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_extras:
        gbs, desc, threads, _ = oracle_sample(cfg, 10.0)  # ~10 s of CPU work (bounded sample)
        cpu = {"value": gbs, "unit": "GB/s", "cores": threads, "kind": "oracle", "sample": desc,
               "cpu_model": cpu_model()}

    value = total_bytes / (ms * 1e-3) / 1e9
    pl = step_main.plan
    line = {
        "metric": METRIC,
        "value": value,
        "unit": "GB/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "us_per_step": ms * 1e3,
        "tokens_per_s": cfg.num_seqs / (ms * 1e-3),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": cfg.dtype,
        "data": "synthetic",
        "config": {
            "workload": cfg.name, "batch": cfg.num_seqs, "q_heads": cfg.num_q_heads,
            "kv_heads": cfg.num_kv_heads, "head_dim": cfg.head_dim,
            "ctx": max(cfg.context_lens), "block_size": cfg.block_size, "tp": world,
            "kernel": KERNEL_NAMES[pl["kernel"]],
            "prefetch": opt_kw.get("prefetch", pda._lib.DEFAULT_PREFETCH),
            "prefetch_distance": opt_kw.get("prefetch_distance", pda._lib.DEFAULT_DISTANCE),
            "smem_stages": pl["smem_stages"], "partition_tokens": pl["partition_tokens"],
            "eviction": ["normal", "demand_first", "prefetch_last", "both"][pl["eviction"]],
            "issue": "self (consumer warps refill their ring stages)" if pl["threads"] == 128 else "producer warp",
            "tp_gather": ("fused into the kernel stores (symmetric memory; first step checked bitwise against NCCL)"
                          if tp_gather == "fused" else "NCCL all_gather_into_tensor"),
            "p_max": pl["p_max"],
            "l2": (f"no flush: inputs larger than L2 ({local_cfg.kv_bytes() / 1e9:.2f} GB KV per step vs 126 MB L2)"
                   if flush_buf is None else
                   "L2 flushed between timed steps (512 MiB write + 256 MiB read, outside the per-step CUDA-event spans)"),
            "bytes_per_step": total_bytes,
        },
        "roofline": {
            "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": load_traffic(cfg.name),
            "kernel": KERNEL_NAMES[pl["kernel"]] + (
                (f" (clusters of {pl['cluster']}, DSMEM merge)" if pl["cluster"] else " + combine_kernel")
                if pl["kernel"] == 2 and pl["p_max"] > 1 else ""),
            "launch_us": attn_ms * 1e3, "algorithmic_bytes_per_launch": local_bytes,
            "peak_source": peak_src,
            # the copy peak counts read + write traffic of a copy; a read-only stream runs
            # faster, so frac > 1 is possible -- context against the spec and the in-run probe:
            "frac_of_spec_8000_gbs": achieved / 8000.0,
            "frac_of_read_probe": (achieved / extras["read_roofline_gbs"]) if "read_roofline_gbs" in extras
            else None,
        },
        "step_us_spread": step_spread.get("step"),
        "attention_us_spread": step_spread.get("attention"),
        "cuda_graph": graph,
        "gpu_launches": args.steps * step_main.launches_per_step(),
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
        "e2e": e2e,
    }
    line.update(extras)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist.is_initialized():
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
