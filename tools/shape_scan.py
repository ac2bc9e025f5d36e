"""Library-default step time over a grid of shapes (planner health check).

    python tools/shape_scan.py [--out gpurun_out/shape_scan.jsonl] [--dtype bf16]

Uniform context lengths; heads (Hq/Hkv) from the paper's model table
(DS7) plus TP shards; batch 1-512; context 1k-32k; cells with more
than 24 GB of KV are skipped.  One JSON line per cell: µs (median of CUDA-graph
replays after a clean L2 flush), algorithmic GB/s, the plan.
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2504_06319_b200 as pda
import synth
from bench import L2Flush

HEADS = [(32, 32), (32, 8), (64, 8), (28, 4), (40, 8), (32, 2), (8, 1), (4, 4), (16, 16)]
BATCH = [1, 8, 32, 128, 512]
CTX = [1024, 8192, 32768]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/shape_scan.jsonl")
    ap.add_argument("--dtype", default="bf16")
    ap.add_argument("--reps", type=int, default=7)
    a = ap.parse_args()
    flush = L2Flush(torch)
    f = open(a.out, "w")
    for hq, hkv in HEADS:
        for B in BATCH:
            for ctx in CTX:
                kv = 2 * B * hkv * ctx * 128 * 2
                if kv > 24e9:
                    continue
                cfg = synth.uniform(f"s_{B}_{hq}_{hkv}_{ctx}", B, hq, hkv, 128, ctx, a.dtype)
                inp = synth.make_inputs(cfg, seed=1, device="cuda", poison=False)
                args = (inp["q"], inp["k_cache"], inp["v_cache"], inp["block_tables"], inp["context_lens"],
                        inp["scale"])
                out = pda.paged_decode_attention(*args)
                ws = torch.zeros(1 << 28, dtype=torch.uint8, device="cuda")
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, capture_error_mode="relaxed"):
                    pda.paged_decode_attention(*args, out=out, workspace=ws)
                spans = []
                for _ in range(a.reps):
                    flush()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    g.replay()
                    e1.record()
                    spans.append((e0, e1))
                torch.cuda.synchronize()
                us = statistics.median(x.elapsed_time(y) * 1e3 for x, y in spans)
                shape = pda.make_shape(inp["q"], inp["k_cache"], inp["block_tables"])
                pl = pda.plan(shape, pda.make_options())
                tot = cfg.kv_bytes() + cfg.other_bytes()
                rec = dict(B=B, hq=hq, hkv=hkv, ctx=ctx, dtype=a.dtype, kv_gb=round(cfg.kv_bytes() / 1e9, 3),
                           us=round(us, 2), gbs=round(tot / us / 1e3), p_max=pl["p_max"],
                           P=pl["partition_tokens"], stages=pl["smem_stages"], cluster=pl["cluster"],
                           ctas=pl["grid_x"] * pl["grid_y"] * pl["grid_z"])
                f.write(json.dumps(rec) + "\n")
                f.flush()
                print(json.dumps(rec), flush=True)
                del inp, args, out, ws, g
                torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
