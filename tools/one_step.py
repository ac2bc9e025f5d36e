"""A few launches of one configuration (for ncu captures): warm-up + 2 more.

    python tools/one_step.py CONFIG ['{options}'] [kv8]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2504_06319_b200 as pda
import synth
from bench import workload_config

cfg = workload_config(sys.argv[1])
kw = eval(sys.argv[2]) if len(sys.argv) > 2 else {}
inp = synth.make_inputs(cfg, seed=1234, device="cuda", shuffle=os.environ.get("PSWEEP_CONTIGUOUS") != "1")
if len(sys.argv) > 3 and sys.argv[3] == "kv8":
    inp = synth.quantize_kv_e4m3(inp)
    kw.update(k_scale=inp["k_scale"], v_scale=inp["v_scale"])
for _ in range(3):
    pda.paged_decode_attention(inp["q"], inp["k_cache"], inp["v_cache"], inp["block_tables"], inp["context_lens"],
                               inp["scale"], **kw)
torch.cuda.synchronize()
