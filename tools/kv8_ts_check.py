"""e4m3 D-split (tile-split) kernel check, for the A/B switch PDA_TILE_SPLIT_KV8:
    PDA_TILE_SPLIT_KV8=1 python tools/kv8_ts_check.py ts     # split kernel: vs the fp64 oracle, outputs saved
    python tools/kv8_ts_check.py pair                        # pair kernel: same shapes, outputs saved
    python tools/kv8_ts_check.py cmp                         # the two bitwise equal?
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2504_06319_b200 as pda
import synth

SHAPES = [
    synth.Config("kv8_mha", 4, 4, 4, 128, (1, 15, 17, 300), "fp16", poison_blocks=5),
    synth.Config("kv8_gqa4_bf16", 3, 16, 4, 128, (100, 1000, 513), "bf16", poison_blocks=3),
    synth.Config("kv8_gqa8", 2, 16, 2, 128, (777, 64), "fp16", poison_blocks=2),
    synth.Config("kv8_zero", 3, 4, 2, 128, (0, 5, 0), "fp16", poison_blocks=1),
    synth.Config("kv8_long", 4, 32, 8, 128, (4096, 3000, 17, 2049), "bf16", poison_blocks=2),
]
mode = sys.argv[1]
path = "/tmp/kv8_ts_{}.pt"
if mode == "cmp":
    a, b = torch.load(path.format("ts")), torch.load(path.format("pair"))
    bad = [k for k in a if not torch.equal(a[k], b[k])]
    print("kv8 split vs pair bitwise:", "OK" if not bad else f"DIFFER {bad}", f"({len(a)} cases)")
    sys.exit(1 if bad else 0)
import oracle  # test infrastructure (this is a check tool)
res, worst = {}, 0.0
for cfg in SHAPES:
    inp = synth.quantize_kv_e4m3(synth.make_inputs(cfg, seed=17), k_scale=1 / 224, v_scale=1 / 256)
    ref = oracle.paged_attention_kv8(inp["q"], inp["k_cache"], inp["v_cache"], inp["k_scale"], inp["v_scale"],
                                     inp["block_tables"], inp["context_lens"], inp["scale"], cfg.dtype)
    dev = {k: (v.cuda() if torch.is_tensor(v) else v) for k, v in inp.items()}
    for st in (16, 24):
        for kw in (dict(), dict(partition_tokens=64)):
            out = pda.paged_decode_attention(dev["q"], dev["k_cache"], dev["v_cache"], dev["block_tables"],
                                             dev["context_lens"], dev["scale"], k_scale=dev["k_scale"],
                                             v_scale=dev["v_scale"], smem_stages=st, prefetch="off", **kw)
            torch.cuda.synchronize()
            err = float(np.abs(out.double().cpu().numpy() - ref).max())
            worst = max(worst, err)
            assert err <= 2e-3, (cfg.name, st, kw, err)
            res[f"{cfg.name}_{st}_{kw}"] = out.cpu()
torch.save(res, path.format(mode))
print(f"kv8 {mode}: {len(res)} cases vs oracle, max abs err {worst:.2e}")
