"""Latency floor of a decode step: per-call time of back-to-back calls
(eager, one event pair over N calls) and of CUDA-graph replays, for small
presets.  python tools/floor.py c4_b1_ctx512 c4_b1_ctx4096 ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2504_06319_b200 as pda
import synth
from bench import workload_config

for name in sys.argv[1:]:
    cfg = workload_config(name)
    inp = synth.make_inputs(cfg, seed=0, device="cuda")
    ws = torch.zeros(64 << 20, dtype=torch.uint8, device="cuda")
    out = pda.paged_decode_attention(inp["q"], inp["k_cache"], inp["v_cache"], inp["block_tables"],
                                     inp["context_lens"], inp["scale"], workspace=ws)

    def call():
        pda.paged_decode_attention(inp["q"], inp["k_cache"], inp["v_cache"], inp["block_tables"],
                                   inp["context_lens"], inp["scale"], out=out, workspace=ws)
    for _ in range(10):
        call()
    torch.cuda.synchronize()
    n = 200
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        call()
    b.record()
    torch.cuda.synchronize()
    eager = a.elapsed_time(b) / n * 1e3
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(20):
            call()
    g.replay()
    torch.cuda.synchronize()
    a.record()
    for _ in range(10):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    graph = a.elapsed_time(b) / 200 * 1e3
    print(f"{name}: back-to-back eager {eager:.2f} us/call, graph of 20 calls {graph:.2f} us/call "
          f"(L2-warm: KV {cfg.kv_bytes() / 1e6:.1f} MB)")
