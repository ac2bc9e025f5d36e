"""tcgen05 kernel: parity vs the fp64 oracle on small shapes, then timings
against split-K on bench / sweep cells (CUDA-graph replays, L2 flushed).

    python tools/tc_check.py [parity|time|all]
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
import paper_2504_06319_b200 as pda
import synth
from bench import L2Flush, workload_config

MODE = sys.argv[1] if len(sys.argv) > 1 else "all"


def run(inp, **kw):
    return pda.paged_decode_attention(inp["q"], inp["k_cache"], inp["v_cache"], inp["block_tables"],
                                      inp["context_lens"], inp["scale"], prefetch="off", **kw)


if MODE in ("parity", "all"):
    shapes = [
        synth.Config("t_mha", 2, 4, 4, 128, (128, 300), "fp16", poison_blocks=2),
        synth.Config("t_gqa8_bf16", 3, 16, 2, 128, (777, 64, 1), "bf16", poison_blocks=2),
        synth.Config("t_gqa16", 2, 32, 2, 128, (95, 2500), "fp16", poison_blocks=2),
        synth.Config("t_gqa4_bf16", 5, 16, 4, 128, (100, 1000, 0, 513, 16), "bf16", poison_blocks=3),
        synth.Config("t_long", 1, 8, 1, 128, (9000,), "bf16", poison_blocks=1),
    ]
    for cfg in shapes:
        for kw in (dict(kernel="tc"), dict(kernel="tc", num_sms=3), dict(kernel="tc", num_sms=1)):
            inp = synth.make_inputs(cfg, seed=3)
            dev = {k: (v.cuda() if torch.is_tensor(v) else v) for k, v in inp.items()}
            try:
                out = run(dev, **kw)
                torch.cuda.synchronize()
            except Exception as e:  # noqa: BLE001
                print(json.dumps(dict(cfg=cfg.name, kw=kw, error=str(e)[:200])), flush=True)
                continue
            ref = oracle.paged_attention(inp["q"], inp["k_cache"], inp["v_cache"], inp["block_tables"],
                                         inp["context_lens"], inp["scale"], cfg.dtype)
            g = out.double().cpu().numpy()
            err = float(np.nanmax(np.abs(g - ref))) if np.isfinite(g).all() else float("nan")
            print(json.dumps(dict(cfg=cfg.name, kw=kw, max_err=err, ok=bool(err <= 2e-3))), flush=True)

if MODE in ("time", "all"):
    flush = L2Flush(torch)
    ws = torch.zeros(1 << 28, dtype=torch.uint8, device="cuda")
    for name in ["u_128_8_1_128_8192_bf16", "u_128_32_2_128_8192_bf16", "c4_b64_ctx4096", "c4_b16_ctx4096",
                 "c4_b4_ctx32768", "c2", "c3", "c4_b256_ctx4096"]:
        cfg = workload_config(name)
        inp = synth.make_inputs(cfg, seed=0, device="cuda")
        res = {}
        for label, kw in (("splitk", dict()), ("tc", dict(kernel="tc"))):
            out = run(inp, workspace=ws, **kw)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, capture_error_mode="relaxed"):
                run(inp, out=out, workspace=ws, **kw)
            ts = []
            for _ in range(10):
                flush()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(); g.replay(); e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e3)
            res[label] = statistics.median(ts)
        a = run(inp, workspace=ws)
        b = run(inp, workspace=ws, kernel="tc")
        diff = float((a.float() - b.float()).abs().max())
        tot = cfg.kv_bytes() + cfg.other_bytes()
        print(json.dumps(dict(cell=name, splitk_us=round(res["splitk"], 2), tc_us=round(res["tc"], 2),
                              splitk_gbs=round(tot / res["splitk"] / 1e3), tc_gbs=round(tot / res["tc"] / 1e3),
                              max_diff_vs_splitk=diff)), flush=True)
        del inp
