"""Per-tile event times of the tc kernel (a PDA_TC_STAMPS=1 build via PDA_LIB_PATH).

    PDA_LIB_PATH=build_ab/tc_stamps/libpda.so python tools/tc_stamps.py CELL [l2]

Events (clock64 on the CTA's SM): 0 K issued, 1 V issued, 2 QK^T issued,
3 S seen by the softmax group, 4 P written, 5 PV issued.  Prints medians over
CTAs x tiles (steady tiles 8..63) of the intervals between them, in cycles.
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2504_06319_b200 as pda
import synth
from bench import workload_config

cfg = workload_config(sys.argv[1])
l2 = len(sys.argv) > 2 and sys.argv[2] == "l2"
inp = synth.make_inputs(cfg, seed=0, device="cuda")
bt = inp["block_tables"]
if l2:
    slab = cfg.num_kv_heads * 16 * cfg.head_dim * 4
    bt = (bt % max(1, int(48e6 / slab))).contiguous()
shape = pda.make_shape(inp["q"], inp["k_cache"], bt)
opts = pda.make_options(kernel="tc", prefetch="off")
info = pda.plan(shape, opts)
ws = torch.zeros(info["workspace_bytes"], dtype=torch.uint8, device="cuda")
for _ in range(3):
    pda.paged_decode_attention(inp["q"], inp["k_cache"], inp["v_cache"], bt, inp["context_lens"], inp["scale"],
                               kernel="tc", prefetch="off", workspace=ws)
torch.cuda.synchronize()
G, nh, B = info["grid_x"], (8 if cfg.num_q_heads // cfg.num_kv_heads <= 8 else 16), cfg.num_seqs
a256 = lambda x: (x + 255) // 256 * 256
off = a256(G * 2 * nh * 128 * 4) + a256(G * 2 * nh * 4) + (B + 1) * 8
st = ws[off:off + G * 64 * 8 * 8].view(torch.int64).view(G, 64, 8).cpu().numpy().astype(np.float64)
ev = {}
names = ["K", "V", "QK", "S", "P", "PV"]
pairs = [("K", "QK"), ("QK", "S"), ("S", "P"), ("P", "PV"), ("V", "PV"), ("K", "V")]
res = {}
for a, b in pairs:
    ia, ib = names.index(a), names.index(b)
    d = st[:, 8:, ib] - st[:, 8:, ia]
    res[f"{a}->{b}"] = float(np.median(d))
for name in names:  # per-tile period of each event
    i = names.index(name)
    res[f"period_{name}"] = float(np.median(np.diff(st[:, 8:, i], axis=1)))
print(json.dumps(dict(cell=cfg.name, l2=l2, cycles=res)))
