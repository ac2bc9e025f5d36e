"""One launch of a kernel variant on a sweep cell (c4_b{B}_ctx{C}) or preset (debug aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2504_06319_b200 as pda
import synth
from bench import workload_config

kw = eval(sys.argv[1])
cfg = workload_config(sys.argv[2])
inp = synth.make_inputs(cfg, seed=0, device="cuda")
for _ in range(int(sys.argv[3]) if len(sys.argv) > 3 else 2):
    out = pda.paged_decode_attention(inp["q"], inp["k_cache"], inp["v_cache"], inp["block_tables"],
                                     inp["context_lens"], inp["scale"], **kw)
torch.cuda.synchronize()
print("ok", kw, sys.argv[2])
