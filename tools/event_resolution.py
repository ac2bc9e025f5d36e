"""Probe the CUDA-event timer resolution on this GPU (per-call spans of a
short kernel): prints the distinct elapsed times seen."""
import torch

x = torch.zeros(1 << 20, device="cuda")
spans = []
for _ in range(200):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        x.add_(1)
    b.record()
    spans.append((a, b))
torch.cuda.synchronize()
vals = sorted(set(round(a.elapsed_time(b) * 1e3, 3) for a, b in spans))
print("distinct us:", vals[:40])
