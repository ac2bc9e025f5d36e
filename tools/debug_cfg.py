"""Run one kernel variant on a synthetic config given as B,Hq,Hkv,D,ctx,dtype (debug aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2504_06319_b200 as pda
import synth

kw = eval(sys.argv[1]) if len(sys.argv) > 1 else {}
B, Hq, Hkv, D, ctx, dt = sys.argv[2].split(",")
cfg = synth.uniform("dbg", int(B), int(Hq), int(Hkv), int(D), int(ctx), dt)
inp = synth.make_inputs(cfg, seed=0, device="cuda")
out = pda.paged_decode_attention(inp["q"], inp["k_cache"], inp["v_cache"], inp["block_tables"],
                                 inp["context_lens"], inp["scale"], **kw)
torch.cuda.synchronize()
print("ok", kw, sys.argv[2], out.float().abs().max().item(), torch.isfinite(out).all().item())
