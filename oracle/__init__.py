"""fp64 CPU oracle for paged decode attention -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (``paper_2504_06319_b200``) never imports it, and this package
imports nothing from the product.  The arithmetic lives in ``oracle.c``
(plain C, fp64, OpenMP over output rows); this module only marshals numpy
arrays into it.

Citations are to /root/reference/PAPER.md lines (P:n); see oracle.c for the
per-function citations and DESIGN.md section "Oracle" for the pins.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

DTYPES = {"fp16": 0, "bf16": 1}


def build(force: bool = False) -> str:
    """Compile oracle.c into liboracle.so with gcc (-O2, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11", _SRC, "-o", _LIB, "-lm"]
        subprocess.check_call(cmd)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB)
            p = ctypes.c_void_p
            i32, i64, f64 = ctypes.c_int, ctypes.c_int64, ctypes.c_double
            L.oracle_fp16_to_f64.argtypes = [ctypes.c_uint16]
            L.oracle_fp16_to_f64.restype = f64
            L.oracle_bf16_to_f64.argtypes = [ctypes.c_uint16]
            L.oracle_bf16_to_f64.restype = f64
            L.oracle_paged_attention.argtypes = [p, p, p, i32, p, p, i32, i32, i32, i32, i32, i32,
                                                 f64, p, p, i64, i32]
            L.oracle_paged_attention.restype = i32
            L.oracle_attention_weights.argtypes = [p, p, i32, p, p, i32, i32, i32, i32, i32, i32,
                                                   i32, f64, p]
            L.oracle_attention_weights.restype = i32
            L.oracle_plan_splitk.argtypes = [p, p, i32, i32, i32, i32, i32, i32, i32, p]
            L.oracle_plan_splitk.restype = i32
            L.oracle_plan_paper.argtypes = [p, p, i32, i32, i32, i32, i32, i32, p]
            L.oracle_plan_paper.restype = i32
            L.oracle_plan_stream.argtypes = [p, p, i32, i32, i32, i32, i32, i32, p]
            L.oracle_plan_stream.restype = i32
            L.oracle_e4m3_to_f64.argtypes = [ctypes.c_uint8]
            L.oracle_e4m3_to_f64.restype = f64
            L.oracle_paged_attention_kv8.argtypes = [p, i32, p, p, f64, f64, p, p, i32, i32, i32, i32,
                                                     i32, i32, f64, p, p, i64, i32]
            L.oracle_paged_attention_kv8.restype = i32
            L.oracle_paged_attention_mq.argtypes = [p, p, p, i32, p, p, i32, i32, i32, i32, i32, i32,
                                                    i32, f64, p, i32]
            L.oracle_paged_attention_mq.restype = i32
            L.oracle_eq1_block_bytes.argtypes = [i64, i64, i64]
            L.oracle_eq1_block_bytes.restype = i64
            L.oracle_eq2_total_bytes.argtypes = [i64, i64, i64, i64]
            L.oracle_eq2_total_bytes.restype = i64
            L.oracle_l2_residency_bound.argtypes = [i64, i64]
            L.oracle_l2_residency_bound.restype = i64
            L.oracle_max_threads.restype = i32
            L.oracle_validate_inputs.argtypes = [p, p, i32, i32, i32, i64, p]
            L.oracle_validate_inputs.restype = i32
            L.oracle_e4m3_encode.argtypes = [ctypes.c_float]
            L.oracle_e4m3_encode.restype = ctypes.c_uint8
            L.oracle_kv_append.argtypes = [p, p, p, p, p, p, i32, i32, i32, i32, i32, i32]
            L.oracle_kv_append.restype = i32
            L.oracle_kv_append_e4m3.argtypes = [p, p, i32, ctypes.c_float, ctypes.c_float, p, p, p, p, i32,
                                                i32, i32, i32, i32, i32]
            L.oracle_kv_append_e4m3.restype = i32
            _lib = L
    return _lib


def _u16(a) -> np.ndarray:
    """Raw 16-bit patterns of an fp16/bf16 array (numpy uint16/float16 or torch tensor)."""
    if hasattr(a, "detach"):  # torch tensor: reinterpret bits without importing torch here
        import torch
        a = a.detach().cpu().contiguous().view(torch.int16).numpy()
    a = np.ascontiguousarray(a)
    return a.view(np.uint16)


def _i32(a) -> np.ndarray:
    if hasattr(a, "detach"):
        a = a.detach().cpu().numpy()
    return np.ascontiguousarray(a, dtype=np.int32)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def paged_attention(q, k_cache, v_cache, block_tables, context_lens, scale: float, dtype: str,
                    rows=None, nthreads: int = 0) -> np.ndarray:
    """fp64 paged decode attention, the plain definition (Oracle).

    q [B, Hq, D], k_cache/v_cache [num_blocks, Hkv, bs, D] (fp16/bf16 bit
    patterns), block_tables [B, max_blocks] int32, context_lens [B] int32.
    Returns out [B, Hq, D] float64 (rows not in ``rows`` are NaN).
    """
    qa, ka, va = _u16(q), _u16(k_cache), _u16(v_cache)
    bt, lens = _i32(block_tables), _i32(context_lens)
    B, Hq, D = qa.shape
    _, Hkv, bs, D2 = ka.shape
    assert D2 == D and va.shape == ka.shape and bt.shape[0] == B and lens.shape == (B,)
    out = np.full((B, Hq, D), np.nan, dtype=np.float64)
    rows_a = None
    n_rows = 0
    if rows is not None:
        rows_a = np.ascontiguousarray(rows, dtype=np.int64)
        n_rows = rows_a.size
    rc = lib().oracle_paged_attention(
        _ptr(qa), _ptr(ka), _ptr(va), DTYPES[dtype], _ptr(bt), _ptr(lens), B, Hq, Hkv, D, bs,
        bt.shape[1], float(scale), _ptr(out), _ptr(rows_a) if rows_a is not None else None,
        n_rows, int(nthreads))
    if rc != 0:
        raise ValueError("oracle_paged_attention: invalid arguments")
    return out


def attention_weights(q, k_cache, block_tables, context_lens, b: int, h: int, scale: float,
                      dtype: str) -> np.ndarray:
    """Softmax weights of row (b, h) over its context tokens, fp64."""
    qa, ka = _u16(q), _u16(k_cache)
    bt, lens = _i32(block_tables), _i32(context_lens)
    B, Hq, D = qa.shape
    _, Hkv, bs, _ = ka.shape
    w = np.zeros(max(1, bt.shape[1] * bs), dtype=np.float64)
    n = lib().oracle_attention_weights(_ptr(qa), _ptr(ka), DTYPES[dtype], _ptr(bt), _ptr(lens),
                                       b, h, Hq, Hkv, D, bs, bt.shape[1], float(scale), _ptr(w))
    return w[:n].copy()


def plan_splitk(block_tables, context_lens, num_kv_heads: int, block_size: int,
                partition_tokens: int, p_max: int, prefetch_distance: int) -> np.ndarray:
    """Per-unit bookkeeping records [B, Hkv, P_max, 4 + 2R] (see oracle.c)."""
    bt, lens = _i32(block_tables), _i32(context_lens)
    B, max_blocks = bt.shape
    R = partition_tokens // block_size
    recs = np.empty((B, num_kv_heads, p_max, 4 + 2 * R), dtype=np.int32)
    rc = lib().oracle_plan_splitk(_ptr(bt), _ptr(lens), B, num_kv_heads, block_size, max_blocks,
                                  partition_tokens, p_max, prefetch_distance, _ptr(recs))
    if rc != 0:
        raise ValueError("oracle_plan_splitk: invalid arguments")
    return recs


def plan_paper(block_tables, context_lens, num_q_heads: int, block_size: int, warps: int,
               prefetch_distance: int) -> np.ndarray:
    """Per-(b, h, warp) Alg. 1 records [B, Hq, w, 4 + 2R], R = ceil(max_blocks / w)."""
    bt, lens = _i32(block_tables), _i32(context_lens)
    B, max_blocks = bt.shape
    R = (max_blocks + warps - 1) // warps
    recs = np.empty((B, num_q_heads, warps, 4 + 2 * R), dtype=np.int32)
    rc = lib().oracle_plan_paper(_ptr(bt), _ptr(lens), B, num_q_heads, block_size, max_blocks,
                                 warps, prefetch_distance, _ptr(recs))
    if rc != 0:
        raise ValueError("oracle_plan_paper: invalid arguments")
    return recs


def plan_stream(block_tables, context_lens, num_kv_heads: int, block_size: int, num_streams: int,
                prefetch_distance: int) -> np.ndarray:
    """Per-row records [B, Hkv, 4 + 2 * max_blocks] of the balanced stream partition."""
    bt, lens = _i32(block_tables), _i32(context_lens)
    B, max_blocks = bt.shape
    recs = np.empty((B, num_kv_heads, 4 + 2 * max_blocks), dtype=np.int32)
    rc = lib().oracle_plan_stream(_ptr(bt), _ptr(lens), B, num_kv_heads, block_size, max_blocks,
                                  num_streams, prefetch_distance, _ptr(recs))
    if rc != 0:
        raise ValueError("oracle_plan_stream: invalid arguments")
    return recs


def _u8(a) -> np.ndarray:
    if hasattr(a, "detach"):
        import torch
        a = a.detach().cpu().contiguous().view(torch.uint8).numpy()
    return np.ascontiguousarray(a).view(np.uint8)


def paged_attention_kv8(q, k_cache, v_cache, k_scale: float, v_scale: float, block_tables,
                        context_lens, scale: float, q_dtype: str, rows=None, nthreads: int = 0):
    """fp64 paged decode attention over an e4m3 KV cache with per-tensor scales."""
    qa, ka, va = _u16(q), _u8(k_cache), _u8(v_cache)
    bt, lens = _i32(block_tables), _i32(context_lens)
    B, Hq, D = qa.shape
    _, Hkv, bs, D2 = ka.shape
    assert D2 == D and va.shape == ka.shape
    out = np.full((B, Hq, D), np.nan, dtype=np.float64)
    rows_a = np.ascontiguousarray(rows, dtype=np.int64) if rows is not None else None
    rc = lib().oracle_paged_attention_kv8(
        _ptr(qa), DTYPES[q_dtype], _ptr(ka), _ptr(va), float(k_scale), float(v_scale), _ptr(bt),
        _ptr(lens), B, Hq, Hkv, D, bs, bt.shape[1], float(scale), _ptr(out),
        _ptr(rows_a) if rows_a is not None else None, rows_a.size if rows_a is not None else 0,
        int(nthreads))
    if rc != 0:
        raise ValueError("oracle_paged_attention_kv8: invalid arguments")
    return out


def paged_attention_mq(q, k_cache, v_cache, block_tables, context_lens, scale: float, dtype: str,
                       nthreads: int = 0) -> np.ndarray:
    """Multi-token causal decode: q [B, q_len, Hq, D] -> out [B, q_len, Hq, D] fp64."""
    qa, ka, va = _u16(q), _u16(k_cache), _u16(v_cache)
    bt, lens = _i32(block_tables), _i32(context_lens)
    B, q_len, Hq, D = qa.shape
    _, Hkv, bs, _ = ka.shape
    out = np.full((B, q_len, Hq, D), np.nan, dtype=np.float64)
    rc = lib().oracle_paged_attention_mq(_ptr(qa), _ptr(ka), _ptr(va), DTYPES[dtype], _ptr(bt), _ptr(lens), B,
                                         q_len, Hq, Hkv, D, bs, bt.shape[1], float(scale), _ptr(out),
                                         int(nthreads))
    if rc != 0:
        raise ValueError("oracle_paged_attention_mq: invalid arguments")
    return out


def e4m3_to_f64(code: int) -> float:
    return lib().oracle_e4m3_to_f64(code)


def fp16_to_f64(bits: int) -> float:
    return lib().oracle_fp16_to_f64(bits)


def bf16_to_f64(bits: int) -> float:
    return lib().oracle_bf16_to_f64(bits)


def eq1_block_bytes(b: int, d_h: int, t_block: int) -> int:
    return lib().oracle_eq1_block_bytes(b, d_h, t_block)


def eq2_total_bytes(m_block: int, n_thread: int, h: int, batch: int) -> int:
    return lib().oracle_eq2_total_bytes(m_block, n_thread, h, batch)


def l2_residency_bound(l2_bytes: int, m_total_b1: int) -> int:
    return lib().oracle_l2_residency_bound(l2_bytes, m_total_b1)


def max_threads() -> int:
    return lib().oracle_max_threads()


def validate_inputs(block_tables, context_lens, num_blocks: int, block_size: int = 16):
    """(sequences with an invalid length, referenced block ids out of range, invalid sequences)."""
    bt, lens = _i32(block_tables), _i32(context_lens)
    counts = np.zeros(3, dtype=np.int64)
    lib().oracle_validate_inputs(_ptr(bt), _ptr(lens), lens.shape[0], bt.shape[1], block_size, int(num_blocks),
                                 _ptr(counts))
    return tuple(int(c) for c in counts)


def e4m3_encode(x: float) -> int:
    """fp32 value -> e4m3 code (nearest, ties to even, saturating, NaN -> 0x7F)."""
    return int(lib().oracle_e4m3_encode(float(x)))


def kv_append(k_new, v_new, k_cache, v_cache, block_tables, context_lens):
    """Return copies of the 16-bit caches with the new rows [B, q_len, Hkv, D] written in place."""
    kn, vn = _u16(k_new), _u16(v_new)
    kc, vc = _u16(k_cache).copy(), _u16(v_cache).copy()
    bt, lens = _i32(block_tables), _i32(context_lens)
    B, q_len, Hkv, D = kn.shape
    bs = kc.shape[2]
    rc = lib().oracle_kv_append(_ptr(kn), _ptr(vn), _ptr(kc), _ptr(vc), _ptr(bt), _ptr(lens), B, q_len, Hkv, D,
                                bs, bt.shape[1])
    if rc != 0:
        raise ValueError("oracle_kv_append: invalid arguments")
    return kc, vc


def kv_append_e4m3(k_new, v_new, dtype: str, k_scale: float, v_scale: float, k_cache, v_cache, block_tables,
                   context_lens):
    """Return copies of the e4m3 caches with the quantised new rows written in place."""
    kn, vn = _u16(k_new), _u16(v_new)
    kc, vc = _u8(k_cache).copy(), _u8(v_cache).copy()
    bt, lens = _i32(block_tables), _i32(context_lens)
    B, q_len, Hkv, D = kn.shape
    bs = kc.shape[2]
    rc = lib().oracle_kv_append_e4m3(_ptr(kn), _ptr(vn), DTYPES[dtype], float(k_scale), float(v_scale), _ptr(kc),
                                     _ptr(vc), _ptr(bt), _ptr(lens), B, q_len, Hkv, D, bs, bt.shape[1])
    if rc != 0:
        raise ValueError("oracle_kv_append_e4m3: invalid arguments")
    return kc, vc
