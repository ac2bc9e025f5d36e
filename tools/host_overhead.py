"""Host-side cost of one decode call (c1 preset): the Python wrapper, the
cached TP step object, and the bare C-ABI call with prebuilt structs."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2504_06319_b200 as pda
from paper_2504_06319_b200 import _lib
from paper_2504_06319_b200.tp import TPDecodeAttention
import synth

inp = synth.make_inputs(synth.C1_TINY, seed=0, device="cuda")
q, k, v, bt, lens, sc = inp["q"], inp["k_cache"], inp["v_cache"], inp["block_tables"], inp["context_lens"], inp["scale"]
out = torch.empty_like(q)
ws = torch.zeros(1 << 20, dtype=torch.uint8, device="cuda")
step = TPDecodeAttention(k, v, 2, 4, bt.shape[1], q.dtype)
shape = _lib.make_shape(q, k, bt)
opts = _lib.make_options()
L = _lib.lib()
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
args = (q.data_ptr(), k.data_ptr(), v.data_ptr(), bt.data_ptr(), lens.data_ptr(), float(sc), out.data_ptr(),
        ctypes.byref(shape), ctypes.byref(opts), ws.data_ptr(), ws.numel(), s)


def bench(fn, n=2000):
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(n):
        fn()
    el = time.perf_counter() - t
    torch.cuda.synchronize()
    return el / n * 1e6


print(f"python wrapper: {bench(lambda: pda.paged_decode_attention(q, k, v, bt, lens, sc, out=out, workspace=ws)):.1f} us/call (host)")
print(f"TP step object: {bench(lambda: step(q, bt, lens, sc)):.1f} us/call (host)")
prep = pda.PreparedDecode(q, k, bt)
print(f"PreparedDecode: {bench(lambda: prep(q, k, v, bt, lens, sc)):.1f} us/call (host)")
print(f"bare C ABI    : {bench(lambda: L.paged_decode_attention(*args)):.1f} us/call (host)")
print(f"plan only     : {bench(lambda: L.pda_plan(ctypes.byref(shape), ctypes.byref(opts), ctypes.byref(_lib.PlanInfo()))):.1f} us/call")
