"""Where does the paper's L2 prefetch pay?  Interleaved A/B with spreads.

For each cell, every variant is captured once in a CUDA graph; then ROUNDS
rounds replay each variant once (L2 flushed before every replay, the variant
order rotated per round), timed with CUDA events.  Printed per cell and
variant: median / p10 / p90 step time, and the paired speedup over the
baseline variant (same round) with its p10 / p90 -- a speedup whose p10 is
above 1 wins in at least 90 % of the rounds.

    python tools/prefetch_policy_ab.py [ROUNDS] CELL [CELL ...]
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2504_06319_b200 as pda
import synth
from bench import L2Flush, spread, workload_config

VARIANTS = [
    ("splitk off", dict()),
    ("splitk line d4", dict(prefetch="line", prefetch_distance=4)),
    ("splitk bulk d4", dict(prefetch="bulk", prefetch_distance=4)),
    ("paper off", dict(kernel="paper")),
    ("paper bulk d4", dict(kernel="paper", prefetch="bulk", prefetch_distance=4)),
    ("paper bulk d4 evict_last", dict(kernel="paper", prefetch="bulk", prefetch_distance=4,
                                      eviction="prefetch_last")),
    ("paper line d4 evict_last", dict(kernel="paper", prefetch="line", prefetch_distance=4,
                                      eviction="prefetch_last")),
]


def main():
    args = sys.argv[1:]
    rounds = int(args.pop(0)) if args and args[0].isdigit() else 50
    flush = L2Flush(torch)
    ws = torch.zeros(1 << 28, dtype=torch.uint8, device="cuda")
    for name in args:
        cfg = workload_config(name)
        inp = synth.make_inputs(cfg, seed=0, device="cuda")
        a = (inp["q"], inp["k_cache"], inp["v_cache"], inp["block_tables"], inp["context_lens"], inp["scale"])
        graphs = []
        for label, kw in VARIANTS:
            out = pda.paged_decode_attention(*a, workspace=ws, **kw)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, capture_error_mode="relaxed"):
                pda.paged_decode_attention(*a, out=out, workspace=ws, **kw)
            graphs.append(g)
        times = [[] for _ in VARIANTS]
        for r in range(rounds):
            order = [(r + i) % len(VARIANTS) for i in range(len(VARIANTS))]
            ev = []
            for i in order:
                flush()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                graphs[i].replay()
                e1.record()
                ev.append((i, e0, e1))
            torch.cuda.synchronize()
            for i, e0, e1 in ev:
                times[i].append(e0.elapsed_time(e1) * 1e3)
        base_off = {"splitk": times[0], "paper": times[3]}
        best = min(range(len(VARIANTS)), key=lambda i: statistics.median(times[i]))
        for i, (label, kw) in enumerate(VARIANTS):
            fam = label.split()[0]
            sp = [b / t for b, t in zip(base_off[fam], times[i])]
            vs_prod = [b / t for b, t in zip(times[0], times[i])]
            print(json.dumps(dict(cell=name, variant=label, us=spread(times[i]),
                                  speedup_vs_same_kernel_off=spread(sp), speedup_vs_splitk_off=spread(vs_prod),
                                  best=i == best, kv_mb=round(cfg.kv_bytes() / 1e6, 1))), flush=True)
        del inp, graphs


if __name__ == "__main__":
    main()
