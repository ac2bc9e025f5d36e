"""Partition-size / ring-depth sweep for one config (CUDA-graph replays, L2 flushed)."""
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
variants = eval(sys.argv[2])
kv8 = len(sys.argv) > 3 and sys.argv[3] == "kv8"
q_len = int(sys.argv[4]) if len(sys.argv) > 4 else 1
# PSWEEP_CONTIGUOUS=1: identity block placement (sequential KV) instead of the shuffled pool
inp = synth.make_inputs(cfg, seed=0, device="cuda", shuffle=os.environ.get("PSWEEP_CONTIGUOUS") != "1")
if q_len > 1:
    inp = synth.with_query_tokens(inp, q_len)
if kv8:
    inp = synth.quantize_kv_e4m3(inp)
    variants = [dict(v, k_scale=inp["k_scale"], v_scale=inp["v_scale"]) for v in variants]
ws = torch.zeros(1 << 30, dtype=torch.uint8, device="cuda")
flush = L2Flush(torch)
res = {}
graphs = {}
outs = {}
for i, v in enumerate(variants):
    outs[i] = pda.paged_decode_attention(inp["q"], inp["k_cache"], inp["v_cache"], inp["block_tables"],
                                         inp["context_lens"], inp["scale"], workspace=ws, **v)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, capture_error_mode="relaxed"):
        pda.paged_decode_attention(inp["q"], inp["k_cache"], inp["v_cache"], inp["block_tables"],
                                   inp["context_lens"], inp["scale"], out=outs[i], workspace=ws, **v)
    graphs[i] = g
    res[i] = []
for rnd in range(5):
    for i in graphs:
        spans = []
        for _ in range(3):  # all reps queued, one sync: no host gaps inside a span
            flush()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); graphs[i].replay(); e1.record()
            spans.append((e0, e1))
        torch.cuda.synchronize()
        res[i].extend(e0.elapsed_time(e1) * 1e3 for e0, e1 in spans)
tot = cfg.kv_bytes() // (2 if kv8 else 1) + cfg.other_bytes()
for i, v in enumerate(variants):
    us = statistics.median(res[i])
    print(json.dumps(dict(cell=cfg.name + ("_kv8" if kv8 else "") + (f"_q{q_len}" if q_len > 1 else ""), **v,
                          us=round(us, 2), gbs=round(tot / us / 1e3),
                          tokens_per_s=round(cfg.num_seqs * q_len / us * 1e6))))
