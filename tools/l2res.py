"""Is a cell's per-CTA rate capped by memory or by the consumer chain?

Times a cell twice with CUDA-graph replays: (a) as generated (HBM-resident KV,
L2 flushed before each replay) and (b) with every block-table entry folded
into a small pool of `pool_mb` MB of KV (L2-resident, no flush).  Same grid,
same plan, same instruction stream; only where the bytes come from differs.
If (b) is not much faster than (a), the cap is on the SM side.

    python tools/l2res.py CELL [VARIANTS] [kv8] [pool_mb]
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

cfg = workload_config(sys.argv[1])
variants = eval(sys.argv[2]) if len(sys.argv) > 2 else [dict()]
kv8 = len(sys.argv) > 3 and sys.argv[3] == "kv8"
pool_mb = float(sys.argv[4]) if len(sys.argv) > 4 else 48.0
inp = synth.make_inputs(cfg, seed=0, device="cuda")
if kv8:
    inp = synth.quantize_kv_e4m3(inp)
    variants = [dict(v, k_scale=inp["k_scale"], v_scale=inp["v_scale"]) for v in variants]
slab = cfg.num_kv_heads * cfg.block_size * cfg.head_dim * (1 if kv8 else 2) * 2  # K+V bytes per block
pool = max(1, int(pool_mb * 1e6 / slab))
bt_res = (inp["block_tables"] % pool).contiguous()
ws = torch.zeros(1 << 30, dtype=torch.uint8, device="cuda")
flush = L2Flush(torch)
tot = cfg.kv_bytes() // (2 if kv8 else 1) + cfg.other_bytes()


def timed(bt, do_flush, v):
    out = pda.paged_decode_attention(inp["q"], inp["k_cache"], inp["v_cache"], bt, inp["context_lens"],
                                     inp["scale"], workspace=ws, **v)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, capture_error_mode="relaxed"):
        pda.paged_decode_attention(inp["q"], inp["k_cache"], inp["v_cache"], bt, inp["context_lens"],
                                   inp["scale"], out=out, workspace=ws, **v)
    res = []
    for _ in range(15):
        if do_flush:
            flush()
        else:
            g.replay()  # warm the pool into L2
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record()
        torch.cuda.synchronize()
        res.append(e0.elapsed_time(e1) * 1e3)
    return statistics.median(res)


if os.environ.get("L2RES_ONCE"):  # ncu capture: warm-up + one L2-resident launch per variant, no timing
    for v in variants:
        for _ in range(2):
            pda.paged_decode_attention(inp["q"], inp["k_cache"], inp["v_cache"], bt_res, inp["context_lens"],
                                       inp["scale"], workspace=ws, **v)
    torch.cuda.synchronize()
    sys.exit(0)

for v in variants:
    hbm = timed(inp["block_tables"], True, v)
    l2 = timed(bt_res, False, v)
    print(json.dumps(dict(cell=cfg.name + ("_kv8" if kv8 else ""), **{k: x for k, x in v.items()
                                                                       if k not in ("k_scale", "v_scale")},
                          hbm_us=round(hbm, 2), l2_us=round(l2, 2), hbm_gbs=round(tot / hbm / 1e3),
                          l2_gbs=round(tot / l2 / 1e3), pool_mb=pool_mb)))
