"""ctypes binding of libpda.so (include/pda.h): argument marshalling only.

Every step of the decode path runs in the CUDA kernels behind the C ABI;
this module turns torch tensors into device pointers + the current stream
and turns status codes into exceptions.  There is no fallback: if the
library is missing or a tensor is not on a CUDA device, calls raise.
"""
from __future__ import annotations

import ctypes
import os
import re
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PDA_LIB_PATH") or os.path.join(HERE, "libpda.so")  # override: A/B experiments only
HEADER = os.path.join(os.path.dirname(HERE), "include", "pda.h")

PDA_F16, PDA_BF16, PDA_F32, PDA_E4M3 = 0, 1, 2, 3
PREFETCH = {"off": 0, "none": 0, None: 0, "bulk": 1, "line": 2, "auto": 3}
EVICTION = {"normal": 0, "demand_first": 1, "prefetch_last": 2, "both": 3, "auto": 4}
DEFAULT_EVICTION = "auto"
ISSUE = {"auto": 0, "producer": 1, "self": 2}
KERNEL = {"auto": 0, "paper": 1, "splitk": 2, "stream": 3, "balanced": 4, "tc": 5}

# Product defaults from the round-1 measurements: the TMA ring
# already fetches S blocks ahead into shared memory while the current block is
# computed, so the extra L2 prefetch (the paper's instruction, or per-line) is
# measured 0-9 % slower on every cell with self-issuing consumers -> off by
# default; "line" / "bulk" with a distance remain the ablation switch.
DEFAULT_PREFETCH = "auto"  # planner: the paper kernel + Alg. 1 prefetch on short GQA steps, else off (pda.h)
DEFAULT_DISTANCE = 4


class PdaError(RuntimeError):
    def __init__(self, status: int, what: str):
        super().__init__(f"{what}: {status_string(status)} (status {status})")
        self.status = status


class Shape(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in (
        "num_seqs", "num_q_heads", "num_kv_heads", "head_dim", "block_size", "num_blocks",
        "max_blocks_per_seq", "dtype", "out_dtype", "kv_dtype", "q_len")]


class Options(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in (
        "prefetch", "prefetch_distance", "partition_tokens", "smem_stages", "kernel", "num_sms",
        "stream_warps", "eviction", "issue_mode")] + [("k_scale", ctypes.c_float),
                                                      ("v_scale", ctypes.c_float),
                                                      ("merge", ctypes.c_int32)]


class PlanInfo(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in (
        "kernel", "partition_tokens", "p_max", "smem_stages", "grid_x", "grid_y", "grid_z",
        "threads", "trace_rec_len", "trace_records", "eviction", "cluster")] + [("workspace_bytes", ctypes.c_size_t)]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


_lib = None
_lock = threading.Lock()


def lib():
    """Load libpda.so (raises if it has not been built)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"{LIB_PATH} is missing: build the CUDA extension first "
                    "(python -c 'import __graft_entry__ as g; g.build()')")
            L = ctypes.CDLL(LIB_PATH)
            p, sz, i32, f32 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_float
            ps, po, ppl = ctypes.POINTER(Shape), ctypes.POINTER(Options), ctypes.POINTER(PlanInfo)
            L.pda_check_args.argtypes = [ps, po]
            L.pda_check_args.restype = i32
            L.pda_plan.argtypes = [ps, po, ppl]
            L.pda_plan.restype = i32
            L.pda_workspace_bytes.argtypes = [ps, po]
            L.pda_workspace_bytes.restype = sz
            L.paged_decode_attention.argtypes = [p, p, p, p, p, f32, p, ps, po, p, sz, p]
            L.paged_decode_attention.restype = i32
            L.paged_decode_attention_trace.argtypes = [p, p, p, p, p, f32, p, ps, po, p, sz, p, sz, p]
            L.paged_decode_attention_trace.restype = i32
            L.paged_decode_attention_timeline.argtypes = [p, p, p, p, p, f32, p, ps, po, p, sz, p, sz, p, sz, p]
            L.paged_decode_attention_timeline.restype = i32
            L.paged_decode_attention_gather.argtypes = [p, p, p, p, p, f32, p, i32, i32, i32, ps, po, p, sz, p]
            L.paged_decode_attention_gather.restype = i32
            L.pda_decode_step_host.argtypes = [p, p, p, p, p, p, p, p, p, p, f32, ps, po, p, sz, p]
            L.pda_decode_step_host.restype = i32
            L.pda_kv_append.argtypes = [p, p, p, p, p, p, ps, po, p]
            L.pda_kv_append.restype = i32
            L.paged_decode_attention_append.argtypes = [p, p, p, p, p, p, p, f32, p, ps, po, p, sz, p]
            L.paged_decode_attention_append.restype = i32
            L.pda_validate_inputs.argtypes = [p, p, ps, p, p]
            L.pda_validate_inputs.restype = i32
            L.pda_decode_step_host_async.argtypes = [p, p, p, p, p, p, p, p, p, p, f32, ps, po, p, sz, p, p, p, p]
            L.pda_decode_step_host_async.restype = i32
            L.pda_read_roofline.argtypes = [p, sz, p, p]
            L.pda_read_roofline.restype = i32
            L.pda_read_roofline_mode.argtypes = [p, sz, p, i32, p]
            L.pda_read_roofline_mode.restype = i32
            L.pda_status_string.argtypes = [i32]
            L.pda_status_string.restype = ctypes.c_char_p
            L.pda_abi_version.restype = ctypes.c_int32
            _lib = L
    return _lib


def header_symbols():
    """Function names declared in include/pda.h."""
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w]+\*?\s+\*?(\w+)\(", text, re.M)))


def status_string(status: int) -> str:
    return lib().pda_status_string(int(status)).decode()


def _check(status: int, what: str):
    if status != 0:
        raise PdaError(status, what)


def _dtype_code(dt) -> int:
    import torch
    if dt == torch.float16:
        return PDA_F16
    if dt == torch.bfloat16:
        return PDA_BF16
    if dt == torch.float32:
        return PDA_F32
    if dt in (torch.uint8, torch.float8_e4m3fn):
        return PDA_E4M3
    raise TypeError(f"unsupported dtype {dt}")


def make_shape(q, k_cache, block_tables, out_dtype=None) -> Shape:
    """q [B, Hq, D] (single-token decode) or [B, q_len, Hq, D] (multi-token)."""
    q_len = 1
    if q.dim() == 4:
        B, q_len, Hq, D = q.shape
    else:
        B, Hq, D = q.shape
    nb, Hkv, bs, D2 = k_cache.shape
    if D2 != D:
        raise ValueError("q and k_cache head_dim differ")
    return Shape(B, Hq, Hkv, D, bs, nb, block_tables.shape[1], _dtype_code(q.dtype),
                 _dtype_code(out_dtype if out_dtype is not None else q.dtype), _dtype_code(k_cache.dtype), q_len)


MERGE = {"auto": 0, "combine": 1, "cluster": 2}
OPTION_KEYS = ("prefetch", "prefetch_distance", "partition_tokens", "smem_stages", "kernel", "num_sms",
               "stream_warps", "eviction", "k_scale", "v_scale", "issue_mode", "merge")


def make_options(prefetch=DEFAULT_PREFETCH, prefetch_distance=None, partition_tokens=0,
                 smem_stages=0, kernel="auto", num_sms=0, stream_warps=0,
                 eviction=DEFAULT_EVICTION, k_scale=0.0, v_scale=0.0, issue_mode=0, merge="auto") -> Options:
    mode = PREFETCH[prefetch] if not isinstance(prefetch, int) else prefetch
    if prefetch_distance is None:
        prefetch_distance = DEFAULT_DISTANCE if mode else 0
    kern = KERNEL[kernel] if not isinstance(kernel, int) else kernel
    return Options(mode, int(prefetch_distance), int(partition_tokens), int(smem_stages), kern,
                   int(num_sms), int(stream_warps), int(EVICTION.get(eviction, eviction)),
                   int(ISSUE.get(issue_mode, issue_mode)), float(k_scale), float(v_scale),
                   int(MERGE.get(merge, merge)))


def plan(shape: Shape, opts: Options) -> dict:
    info = PlanInfo()
    _check(lib().pda_plan(ctypes.byref(shape), ctypes.byref(opts), ctypes.byref(info)), "pda_plan")
    return info.as_dict()


def check_args(shape: Shape, opts: Options) -> int:
    return lib().pda_check_args(ctypes.byref(shape), ctypes.byref(opts))


def workspace_bytes(shape: Shape, opts: Options) -> int:
    return lib().pda_workspace_bytes(ctypes.byref(shape), ctypes.byref(opts))


def _require_cuda(*ts):
    for t in ts:
        if not t.is_cuda:
            raise ValueError("paged_decode_attention runs on CUDA tensors only (no CPU path)")
        if not t.is_contiguous():
            raise ValueError("tensors must be contiguous")


def _stream_handle(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def paged_decode_attention(q, k_cache, v_cache, block_tables, context_lens, scale=None, out=None, *,
                           out_dtype=None, prefetch=DEFAULT_PREFETCH, prefetch_distance=None,
                           partition_tokens=0, smem_stages=0, kernel="auto", stream_warps=0,
                           num_sms=0, eviction=DEFAULT_EVICTION, k_scale=0.0, v_scale=0.0,
                           issue_mode=0, merge="auto", workspace=None, stream=None, trace=False, k_new=None,
                           v_new=None, timeline=False):
    """Decode attention over a paged KV cache (see include/pda.h).

    q [B, Hq, D], k_cache/v_cache [num_blocks, Hkv, 16, D] (fp16/bf16 like q, or
    uint8/float8_e4m3fn e4m3 codes dequantised with k_scale / v_scale),
    block_tables [B, max_blocks] int32, context_lens [B] int32, all CUDA.
    k_new/v_new [B, (q_len,) Hkv, D]: append the step's new tokens to the
    caches first (paged_decode_attention_append; fused in the split-K kernel).
    Returns out [B, Hq, D] (and the int32 bookkeeping trace if trace=True;
    timeline=True, split-K only, also returns the per-unit {start ns, end ns,
    SM} uint64 stamps as an int64 tensor [units, 3] -- a measurement export).
    """
    import torch
    _require_cuda(q, k_cache, v_cache, block_tables, context_lens)
    if (k_new is None) != (v_new is None):
        raise ValueError("k_new and v_new go together")
    if k_new is not None:
        _require_cuda(k_new, v_new)
        if trace or timeline:
            raise ValueError("trace and append are separate calls")
        if k_new.dtype != q.dtype or v_new.dtype != q.dtype:
            raise TypeError("k_new / v_new must have q's dtype")
        q_len = q.shape[1] if q.dim() == 4 else 1
        want = q.shape[0] * q_len * k_cache.shape[1] * k_cache.shape[3]
        if k_new.numel() != want or v_new.numel() != want:
            raise ValueError("k_new / v_new must be [B, q_len, Hkv, D]")
    if block_tables.dtype != torch.int32 or context_lens.dtype != torch.int32:
        raise TypeError("block_tables / context_lens must be int32")
    if out is not None:
        out_dtype = out.dtype
    if out_dtype is None and k_cache.dtype in (torch.uint8, torch.float8_e4m3fn):
        out_dtype = q.dtype
    shape = make_shape(q, k_cache, block_tables, out_dtype)
    opts = make_options(prefetch, prefetch_distance, partition_tokens, smem_stages, kernel,
                        num_sms=num_sms, stream_warps=stream_warps, eviction=eviction,
                        k_scale=k_scale, v_scale=v_scale, issue_mode=issue_mode, merge=merge)
    if scale is None:
        scale = q.shape[-1] ** -0.5
    info = plan(shape, opts)
    if out is None:
        out = torch.empty(q.shape, dtype=out_dtype or q.dtype, device=q.device)
    _require_cuda(out)
    wsb = info["workspace_bytes"]
    if wsb and (workspace is None or workspace.numel() * workspace.element_size() < wsb):
        # zero-filled: the stream kernel's arrival tickets must start at 0 (include/pda.h)
        workspace = torch.zeros(wsb, dtype=torch.uint8, device=q.device)
    ws_ptr = workspace.data_ptr() if (workspace is not None and wsb) else None
    s = _stream_handle(stream)
    L = lib()
    if timeline:
        words = info["trace_records"] * info["trace_rec_len"]
        tr = torch.empty(max(1, words), dtype=torch.int32, device=q.device)
        stamps = torch.zeros((max(1, info["trace_records"]), 3), dtype=torch.int64, device=q.device)
        st = L.paged_decode_attention_timeline(
            q.data_ptr(), k_cache.data_ptr(), v_cache.data_ptr(), block_tables.data_ptr(),
            context_lens.data_ptr(), float(scale), out.data_ptr(), ctypes.byref(shape),
            ctypes.byref(opts), ws_ptr, wsb, tr.data_ptr(), words, stamps.data_ptr(), stamps.numel(), s)
        _check(st, "paged_decode_attention_timeline")
        return out, tr, info, stamps
    if trace:
        words = info["trace_records"] * info["trace_rec_len"]
        tr = torch.empty(max(1, words), dtype=torch.int32, device=q.device)
        st = L.paged_decode_attention_trace(
            q.data_ptr(), k_cache.data_ptr(), v_cache.data_ptr(), block_tables.data_ptr(),
            context_lens.data_ptr(), float(scale), out.data_ptr(), ctypes.byref(shape),
            ctypes.byref(opts), ws_ptr, wsb, tr.data_ptr(), words, s)
        _check(st, "paged_decode_attention_trace")
        return out, tr, info
    if k_new is not None:
        st = L.paged_decode_attention_append(
            q.data_ptr(), k_new.data_ptr(), v_new.data_ptr(), k_cache.data_ptr(), v_cache.data_ptr(),
            block_tables.data_ptr(), context_lens.data_ptr(), float(scale), out.data_ptr(), ctypes.byref(shape),
            ctypes.byref(opts), ws_ptr, wsb, s)
        _check(st, "paged_decode_attention_append")
        return out
    st = L.paged_decode_attention(
        q.data_ptr(), k_cache.data_ptr(), v_cache.data_ptr(), block_tables.data_ptr(),
        context_lens.data_ptr(), float(scale), out.data_ptr(), ctypes.byref(shape), ctypes.byref(opts),
        ws_ptr, wsb, s)
    _check(st, "paged_decode_attention")
    return out


def kv_append(k_new, v_new, k_cache, v_cache, block_tables, context_lens, *, k_scale=0.0, v_scale=0.0,
              stream=None):
    """Write the step's new K/V rows [B, (q_len,) Hkv, D] into their paged slots
    (positions context_lens[b] - q_len + i; include/pda.h pda_kv_append)."""
    import torch
    _require_cuda(k_new, v_new, k_cache, v_cache, block_tables, context_lens)
    if k_new.shape != v_new.shape or k_new.dtype != v_new.dtype:
        raise ValueError("k_new / v_new differ")
    if block_tables.dtype != torch.int32 or context_lens.dtype != torch.int32:
        raise TypeError("block_tables / context_lens must be int32")
    q_len = k_new.shape[1] if k_new.dim() == 4 else 1
    B, Hkv, D = k_new.shape[0], k_new.shape[-2], k_new.shape[-1]
    nb, Hkv2, bs, D2 = k_cache.shape
    if (Hkv2, D2) != (Hkv, D):
        raise ValueError("k_new and k_cache disagree on (Hkv, D)")
    shape = Shape(B, Hkv, Hkv, D, bs, nb, block_tables.shape[1], _dtype_code(k_new.dtype),
                  _dtype_code(k_new.dtype), _dtype_code(k_cache.dtype), q_len)
    opts = make_options(k_scale=k_scale, v_scale=v_scale)
    _check(lib().pda_kv_append(k_new.data_ptr(), v_new.data_ptr(), k_cache.data_ptr(), v_cache.data_ptr(),
                               block_tables.data_ptr(), context_lens.data_ptr(), ctypes.byref(shape),
                               ctypes.byref(opts), _stream_handle(stream)), "pda_kv_append")


def validate_inputs(block_tables, context_lens, num_blocks, block_size=16, stream=None):
    """Debug check of device-resident tables/lengths (pda_validate_inputs):
    returns (invalid lengths, out-of-range referenced block ids, invalid sequences)."""
    import torch
    _require_cuda(block_tables, context_lens)
    if block_tables.dtype != torch.int32 or context_lens.dtype != torch.int32:
        raise TypeError("block_tables / context_lens must be int32")
    counts = torch.empty(3, dtype=torch.int64, device=block_tables.device)
    shape = Shape(context_lens.shape[0], 1, 1, 128, block_size, int(num_blocks), block_tables.shape[1],
                  PDA_F16, PDA_F16, PDA_F16, 1)
    _check(lib().pda_validate_inputs(block_tables.data_ptr(), context_lens.data_ptr(), ctypes.byref(shape),
                                     counts.data_ptr(), _stream_handle(stream)), "pda_validate_inputs")
    return tuple(int(c) for c in counts.cpu())


class PreparedDecode:
    """paged_decode_attention with shape, options, plan, workspace and output
    fixed at construction: a call only marshals the data pointers (the
    per-call Python checks of paged_decode_attention cost ~13 us of host time,
    more than a small step's GPU time).  Calls must use tensors of the shapes
    and dtypes given here (checked cheaply: q shape, cache shape).  One
    workspace and one default output per object: calls on several streams at
    once need one object per stream.

    step = PreparedDecode(q, k_cache, block_tables, **options)
    out = step(q, k_cache, v_cache, block_tables, context_lens, scale)
    """

    def __init__(self, q, k_cache, block_tables, out_dtype=None, device=None, **opt_kw):
        import torch
        if k_cache.dtype in (torch.uint8, torch.float8_e4m3fn) and out_dtype is None:
            out_dtype = q.dtype
        self.shape = make_shape(q, k_cache, block_tables, out_dtype)
        self.opts = make_options(**opt_kw)
        self.info = plan(self.shape, self.opts)
        dev = device if device is not None else k_cache.device
        self.wsb = self.info["workspace_bytes"]
        self.ws = torch.zeros(max(1, self.wsb), dtype=torch.uint8, device=dev)  # tickets start at 0
        self._ws_ptr = self.ws.data_ptr() if self.wsb else None
        self.out = torch.empty(tuple(q.shape), dtype=out_dtype or q.dtype, device=dev)
        self._q_shape, self._k_shape = tuple(q.shape), tuple(k_cache.shape)
        self._shape_ref, self._opts_ref = ctypes.byref(self.shape), ctypes.byref(self.opts)
        self._fn = lib().paged_decode_attention

    def __call__(self, q, k_cache, v_cache, block_tables, context_lens, scale, out=None, stream=None):
        if q.shape != self._q_shape or k_cache.shape != self._k_shape:
            raise ValueError("PreparedDecode: tensor shapes differ from the prepared ones")
        o = self.out if out is None else out
        if stream is None:
            import torch
            stream = torch.cuda.current_stream()
        st = self._fn(q.data_ptr(), k_cache.data_ptr(), v_cache.data_ptr(), block_tables.data_ptr(),
                      context_lens.data_ptr(), scale, o.data_ptr(), self._shape_ref, self._opts_ref, self._ws_ptr,
                      self.wsb, stream.cuda_stream)
        if st:
            raise PdaError(st, "paged_decode_attention")
        return o


class GraphedDecode:
    """A decode step captured once into a CUDA graph: replay() re-runs the
    kernels on the static input buffers (q, block_tables, context_lens --
    update them in place) for a few microseconds of host time, whatever the
    step's size.  The caches stay the caller's tensors.

    g = GraphedDecode(PreparedDecode(q, k_cache, bt), q, k_cache, v_cache, bt, lens, scale)
    g.q.copy_(q_next); g.context_lens.add_(1); out = g.replay()
    """

    def __init__(self, prepared, q, k_cache, v_cache, block_tables, context_lens, scale, warmup=2):
        import torch
        self.prepared = prepared
        self.q, self.block_tables, self.context_lens = q.clone(), block_tables.clone(), context_lens.clone()
        self.k, self.v, self.scale = k_cache, v_cache, float(scale)
        side = torch.cuda.Stream(device=q.device)
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):  # warm up (module load, attributes) outside the capture
            for _ in range(warmup):
                self._step()
        torch.cuda.current_stream().wait_stream(side)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.out = self._step()

    def _step(self):
        return self.prepared(self.q, self.k, self.v, self.block_tables, self.context_lens, self.scale)

    def replay(self):
        self.graph.replay()
        return self.out


def paged_decode_attention_gather(q, k_cache, v_cache, block_tables, context_lens, scale, out_peers,
                                  head_offset, total_q_heads, *, out_dtype=None, workspace=None, stream=None,
                                  **opt_kw):
    """Decode step whose stores also perform the TP output all-gather (include/pda.h).

    out_peers: list of device pointers (ints) or CUDA tensors, one per rank, each
    [B, (q_len,) total_q_heads, D]; this rank's heads go to
    [head_offset, head_offset + Hq).  The caller barriers across ranks afterwards.
    """
    import torch
    _require_cuda(q, k_cache, v_cache, block_tables, context_lens)
    ptrs = [t.data_ptr() if hasattr(t, "data_ptr") else int(t) for t in out_peers]
    if out_dtype is None:
        t0 = out_peers[0]
        out_dtype = t0.dtype if hasattr(t0, "dtype") else q.dtype
    shape = make_shape(q, k_cache, block_tables, out_dtype)
    opts = make_options(**opt_kw)
    info = plan(shape, opts)
    wsb = info["workspace_bytes"]
    if wsb and (workspace is None or workspace.numel() * workspace.element_size() < wsb):
        workspace = torch.zeros(wsb, dtype=torch.uint8, device=q.device)
    arr = (ctypes.c_void_p * len(ptrs))(*ptrs)
    st = lib().paged_decode_attention_gather(
        q.data_ptr(), k_cache.data_ptr(), v_cache.data_ptr(), block_tables.data_ptr(), context_lens.data_ptr(),
        float(scale), arr, len(ptrs), int(head_offset), int(total_q_heads), ctypes.byref(shape),
        ctypes.byref(opts), workspace.data_ptr() if wsb else None, wsb, _stream_handle(stream))
    _check(st, "paged_decode_attention_gather")


class HostDecodeStep:
    """End-to-end step from pinned host buffers through pda_decode_step_host:
    H2D of q / block_tables / context_lens, the decode kernel(s) against the
    device-resident caches, D2H of out -- all on one stream per step.

    slots > 1 pipelines consecutive steps through pda_decode_step_host_async:
    step k uses staging slot k % slots (device buffers, pinned host output, a
    copy stream and two events); its copies run on the slot's copy stream and
    overlap the previous step's kernels, which stay in order on the caller's
    (compute) stream.  join(stream) makes `stream` wait for every output copy
    issued so far (call it before reading a result or recording a timer)."""

    def __init__(self, k_cache, v_cache, num_seqs, num_q_heads, max_blocks, dtype, out_dtype=None, slots=1,
                 **opt_kw):
        import torch
        _require_cuda(k_cache, v_cache)
        dev = k_cache.device
        D = k_cache.shape[-1]
        self.k, self.v = k_cache, v_cache
        self.out_dtype = out_dtype or dtype
        self.slots = []
        for _ in range(max(1, int(slots))):
            sl = dict(q_dev=torch.empty((num_seqs, num_q_heads, D), dtype=dtype, device=dev),
                      bt_dev=torch.empty((num_seqs, max_blocks), dtype=torch.int32, device=dev),
                      lens_dev=torch.empty((num_seqs,), dtype=torch.int32, device=dev),
                      out_dev=torch.empty((num_seqs, num_q_heads, D), dtype=self.out_dtype, device=dev))
            sl["out_host"] = torch.empty(sl["out_dev"].shape, dtype=self.out_dtype, pin_memory=True)
            self.slots.append(sl)
        s0 = self.slots[0]
        self.q_dev, self.bt_dev, self.lens_dev, self.out_dev = s0["q_dev"], s0["bt_dev"], s0["lens_dev"], s0["out_dev"]
        self.out_host = s0["out_host"]
        self.shape = make_shape(self.q_dev, k_cache, self.bt_dev, self.out_dtype)
        self.opts = make_options(**opt_kw)
        wsb = workspace_bytes(self.shape, self.opts)
        # one workspace: the kernels of all slots run in order on the compute stream
        self.ws = torch.zeros(max(1, wsb), dtype=torch.uint8, device=dev)
        for sl in self.slots:
            sl["ws"] = self.ws
        self.wsb = wsb
        self.streams = []
        if len(self.slots) > 1:
            for sl in self.slots:
                sl["copy"] = torch.cuda.Stream(device=dev)
                sl["ev_in"], sl["ev_done"] = torch.cuda.Event(), torch.cuda.Event()
                for ev in (sl["ev_in"], sl["ev_done"]):  # create the events now (torch creates on record)
                    ev.record(sl["copy"])
                self.streams.append(sl["copy"])
            torch.cuda.synchronize(dev)
        self.n = 0

    def h2d_bytes(self):
        return sum(t.numel() * t.element_size() for t in (self.q_dev, self.bt_dev, self.lens_dev))

    def d2h_bytes(self):
        return self.out_dev.numel() * self.out_dev.element_size()

    def _run(self, sl, q_host, bt_host, lens_host, scale, stream):
        st = lib().pda_decode_step_host(
            q_host.data_ptr(), bt_host.data_ptr(), lens_host.data_ptr(), sl["out_host"].data_ptr(),
            sl["q_dev"].data_ptr(), sl["bt_dev"].data_ptr(), sl["lens_dev"].data_ptr(),
            sl["out_dev"].data_ptr(), self.k.data_ptr(), self.v.data_ptr(), float(scale),
            ctypes.byref(self.shape), ctypes.byref(self.opts), sl["ws"].data_ptr() if self.wsb else None,
            self.wsb, _stream_handle(stream))
        _check(st, "pda_decode_step_host")
        return sl["out_host"]

    def __call__(self, q_host, bt_host, lens_host, scale, stream=None):
        """Issue one step; returns the pinned host tensor its output lands in
        (valid once the step's stream has been joined / synchronised)."""
        import torch
        if not self.streams:
            return self._run(self.slots[0], q_host, bt_host, lens_host, scale, stream)
        sl = self.slots[self.n % len(self.slots)]
        self.n += 1
        cs = stream if stream is not None else torch.cuda.current_stream()
        st = lib().pda_decode_step_host_async(
            q_host.data_ptr(), bt_host.data_ptr(), lens_host.data_ptr(), sl["out_host"].data_ptr(),
            sl["q_dev"].data_ptr(), sl["bt_dev"].data_ptr(), sl["lens_dev"].data_ptr(),
            sl["out_dev"].data_ptr(), self.k.data_ptr(), self.v.data_ptr(), float(scale),
            ctypes.byref(self.shape), ctypes.byref(self.opts), self.ws.data_ptr() if self.wsb else None,
            self.wsb, ctypes.c_void_p(cs.cuda_stream), ctypes.c_void_p(sl["copy"].cuda_stream),
            ctypes.c_void_p(sl["ev_in"].cuda_event), ctypes.c_void_p(sl["ev_done"].cuda_event))
        _check(st, "pda_decode_step_host_async")
        return sl["out_host"]

    def join(self, stream=None):
        import torch
        caller = stream if stream is not None else torch.cuda.current_stream()
        for s in self.streams:
            caller.wait_stream(s)


READ_PROBE_MODES = {"ldg": 0, "bulk16k": 1, "bulk_ring": 2}


def read_roofline(buf, sink, stream=None, mode="ldg"):
    """Launch the read-only streaming probe over `buf` (CUDA tensor); mode: ldg |
    bulk16k | bulk_ring (include/pda.h pda_read_roofline_mode)."""
    _require_cuda(buf, sink)
    st = lib().pda_read_roofline_mode(buf.data_ptr(), buf.numel() * buf.element_size(), sink.data_ptr(),
                                      READ_PROBE_MODES[mode], _stream_handle(stream))
    _check(st, "pda_read_roofline_mode")
