"""Run each kernel variant once on a tiny config, one process per variant (debug aid)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2504_06319_b200 as pda
kw = eval(sys.argv[1]) if len(sys.argv) > 1 else {}
cfgname = sys.argv[2] if len(sys.argv) > 2 else "c1"
cfg = synth.PRESETS[cfgname]
inp = synth.make_inputs(cfg, seed=0, device="cuda")
out = pda.paged_decode_attention(inp["q"], inp["k_cache"], inp["v_cache"], inp["block_tables"],
                                 inp["context_lens"], inp["scale"], **kw)
torch.cuda.synchronize()
print("ok", kw, out.float().abs().max().item(), torch.isfinite(out).all().item())
