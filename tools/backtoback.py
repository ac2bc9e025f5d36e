"""Steady-state step time of back-to-back decode steps that each read a
different KV cache (as consecutive layers do), no L2 flush needed: R input
sets whose caches together exceed L2 are cycled through a CUDA graph of
R * reps steps; the per-step time is the graph span / steps.  Beside it, the
single flushed step (the bench / shape-scan protocol) of the same cell.  The
difference is the per-step fixed cost (launch, first TMA round trip, drain,
merge) that programmatic dependent launch overlaps with the neighbouring
step in a multi-layer decode.

    python tools/backtoback.py CELL [CELL ...]     (one JSON line per cell)
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2504_06319_b200 as pda
import synth
from bench import L2Flush, workload_config

L2_BYTES = 126 << 20


def main():
    flush = L2Flush(torch)
    for name in sys.argv[1:]:
        cfg = workload_config(name)
        tot = cfg.kv_bytes() + cfg.other_bytes()
        R = max(2, min(8, int(3 * L2_BYTES / cfg.kv_bytes()) + 2))  # >= 3x L2 over the cycle
        sets = [synth.make_inputs(cfg, seed=s, device="cuda") for s in range(R)]
        ws = [torch.zeros(256 << 20, dtype=torch.uint8, device="cuda") for _ in range(R)]
        outs = [pda.paged_decode_attention(i["q"], i["k_cache"], i["v_cache"], i["block_tables"],
                                           i["context_lens"], i["scale"], workspace=w) for i, w in zip(sets, ws)]

        def step(k):
            i = sets[k % R]
            pda.paged_decode_attention(i["q"], i["k_cache"], i["v_cache"], i["block_tables"], i["context_lens"],
                                       i["scale"], out=outs[k % R], workspace=ws[k % R])

        reps = max(2, 24 // R)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, capture_error_mode="relaxed"):
            for k in range(R * reps):
                step(k)
        g1 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g1, capture_error_mode="relaxed"):
            step(0)
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        b2b, single = [], []
        for _ in range(15):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); g.replay(); e1.record()
            torch.cuda.synchronize()
            b2b.append(e0.elapsed_time(e1) * 1e3 / (R * reps))
            flush()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); g1.replay(); e1.record()
            torch.cuda.synchronize()
            single.append(e0.elapsed_time(e1) * 1e3)
        bu, su = statistics.median(b2b), statistics.median(single)
        print(json.dumps(dict(cell=cfg.name, kv_gb=round(cfg.kv_bytes() / 1e9, 3), input_sets=R,
                              steps_per_graph=R * reps, single_flushed_us=round(su, 2),
                              single_gbs=round(tot / su / 1e3), back_to_back_us=round(bu, 2),
                              back_to_back_gbs=round(tot / bu / 1e3),
                              fixed_cost_us=round(su - bu, 2))), flush=True)
        del sets, ws, outs, g, g1
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
