import torch, statistics, json
x = torch.zeros(1, device="cuda")
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    x.add_(1)
for _ in range(10): g.replay()
torch.cuda.synchronize()
r = []
for _ in range(50):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    r.append(e0.elapsed_time(e1) * 1e3)
print(json.dumps(dict(empty_graph_event_us=statistics.median(r), p10=sorted(r)[5], p90=sorted(r)[45])))
