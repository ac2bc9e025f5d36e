"""One e4m3-cache launch of a preset (for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2504_06319_b200 as pda
import synth
from bench import workload_config

cfg = workload_config(sys.argv[1])
kw = eval(sys.argv[2]) if len(sys.argv) > 2 else {}
inp = synth.quantize_kv_e4m3(synth.make_inputs(cfg, seed=0, device="cuda"))
for _ in range(2):
    pda.paged_decode_attention(inp["q"], inp["k_cache"], inp["v_cache"], inp["block_tables"], inp["context_lens"],
                               inp["scale"], k_scale=inp["k_scale"], v_scale=inp["v_scale"], **kw)
torch.cuda.synchronize()
print("ok")
