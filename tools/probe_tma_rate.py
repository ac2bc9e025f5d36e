"""Read-probe rates from HBM and from L2 (a 48 MB buffer re-read): per-SM
TMA / bulk-copy throughput with 1 vs 3 issuing CTAs per SM (pda_read_roofline_mode)."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2504_06319_b200 as pda

sink = torch.zeros(1 << 20, dtype=torch.uint32, device="cuda")
for size in (48 << 20, 4 << 30):
    buf = torch.ones(size, dtype=torch.uint8, device="cuda")
    for mode in ("ldg", "bulk16k", "bulk_ring"):
        for _ in range(3):
            pda.read_roofline(buf, sink, mode=mode)
        ts = []
        for _ in range(20):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); pda.read_roofline(buf, sink, mode=mode); e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        us = statistics.median(ts)
        print(json.dumps(dict(bytes=size, mode=mode, us=round(us, 2), gbs=round(size / us / 1e3))))
    del buf
