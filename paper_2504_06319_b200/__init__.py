"""B200-native paged decode attention with asynchronous L2 KV prefetch
(arXiv 2504.06319's hot path).

The compute lives in libpda.so (hand-written sm_100a CUDA behind the C ABI in
include/pda.h); this package is the thin Python binding plus the
tensor-parallel driver.  Importing the package does not load the library;
the first call does, and raises if it has not been built.
"""
from ._lib import (GraphedDecode, HostDecodeStep, PdaError, PreparedDecode, check_args, header_symbols, kv_append, lib, make_options,
                   make_shape, paged_decode_attention, paged_decode_attention_gather, plan, read_roofline,
                   status_string, validate_inputs, workspace_bytes)

__all__ = ["paged_decode_attention", "PreparedDecode", "GraphedDecode", "paged_decode_attention_gather", "kv_append",
           "validate_inputs",
           "HostDecodeStep", "PdaError", "plan", "workspace_bytes",
           "check_args", "make_shape", "make_options", "read_roofline", "status_string", "lib",
           "header_symbols"]
