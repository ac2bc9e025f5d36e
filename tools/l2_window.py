"""L2 persisting access-policy window as an alternative to prefetch eviction
hints: a window over the leading part of the KV pool with
hitProp = persisting, on the decode stream.  Times back-to-back steps (no L2
flush: the only reuse a window can create is ACROSS steps) and flushed steps,
with and without the window.

    python tools/l2_window.py c2 c4_b16_ctx4096 c4_b4_ctx32768
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from cuda.bindings import runtime as rt

import paper_2504_06319_b200 as pda
import synth
from bench import L2Flush, workload_config


def check(err):
    e = err[0] if isinstance(err, tuple) else err
    if e != rt.cudaError_t.cudaSuccess:
        raise RuntimeError(str(e))


def set_window(stream, base, nbytes, ratio):
    val = rt.cudaStreamAttrValue() if hasattr(rt, "cudaStreamAttrValue") else rt.cudaLaunchAttributeValue()
    w = val.accessPolicyWindow
    w.base_ptr = base
    w.num_bytes = nbytes
    w.hitRatio = ratio
    w.hitProp = rt.cudaAccessProperty.cudaAccessPropertyPersisting
    w.missProp = rt.cudaAccessProperty.cudaAccessPropertyStreaming
    check(rt.cudaStreamSetAttribute(stream.cuda_stream, rt.cudaStreamAttrID.cudaStreamAttributeAccessPolicyWindow
                                    if hasattr(rt.cudaStreamAttrID, "cudaStreamAttributeAccessPolicyWindow")
                                    else rt.cudaLaunchAttributeID.cudaLaunchAttributeAccessPolicyWindow, val))


def main():
    dev = torch.cuda.current_device()
    prop = torch.cuda.get_device_properties(dev)
    err, max_persist = rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrMaxPersistingL2CacheSize, dev)
    err2, max_window = rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrMaxAccessPolicyWindowSize, dev)
    check(rt.cudaDeviceSetLimit(rt.cudaLimit.cudaLimitPersistingL2CacheSize, max_persist))
    flush = L2Flush(torch)
    for name in sys.argv[1:]:
        cfg = workload_config(name)
        inp = synth.make_inputs(cfg, seed=0, device="cuda")
        stream = torch.cuda.Stream()
        res = {}
        with torch.cuda.stream(stream):
            prep = pda.PreparedDecode(inp["q"], inp["k_cache"], inp["block_tables"])

            def step():
                prep(inp["q"], inp["k_cache"], inp["v_cache"], inp["block_tables"], inp["context_lens"],
                     inp["scale"], stream=stream)

            for mode in ("none", "window"):
                if mode == "window":
                    kv = inp["k_cache"].numel() * inp["k_cache"].element_size()
                    nbytes = min(kv, max_window)
                    set_window(stream, inp["k_cache"].data_ptr(), nbytes, min(1.0, max_persist / nbytes))
                for flushed in (False, True):
                    times = []
                    for _ in range(3):
                        step()
                    for _ in range(20):
                        if flushed:
                            flush()
                        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        a.record(stream)
                        step()
                        b.record(stream)
                        times.append((a, b))
                    torch.cuda.synchronize()
                    res[f"{mode}_{'flushed' if flushed else 'back_to_back'}_us"] = statistics.median(
                        x.elapsed_time(y) * 1e3 for x, y in times)
            set_window(stream, 0, 0, 0.0)
            check(rt.cudaCtxResetPersistingL2Cache())
        print(json.dumps(dict(cell=name, kv_bytes=cfg.kv_bytes(), max_persisting_l2=max_persist,
                              max_window=max_window, **{k: round(v, 1) for k, v in res.items()})), flush=True)


if __name__ == "__main__":
    main()
