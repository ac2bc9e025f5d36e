"""Prefetch ablation sweep (BASELINE configs[2]/[3]): batch x context x kernel x
ring depth x prefetch mode/distance, on one B200.

    python tools/sweep.py --out gpurun_out/sweep.jsonl [--quick]

Every variant of a cell runs on the same inputs; variants are interleaved in
rounds (ABAB...) and each timed iteration is preceded by an L2 flush (a
512 MiB memset, then a 256 MiB read so no dirty lines are left for the step
to write back; untimed) so small cells do not run out of L2.  Times are
CUDA-event medians per iteration.  One JSON line per (cell, variant).
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def variants(quick):
    vs = []
    stages = [4, 8] if quick else [4, 8, 12]
    dists = [2, 8] if quick else [1, 2, 4, 8, 16, 32]
    vs.append(dict(kernel="splitk", prefetch="off"))  # the library default (planner-chosen ring depth)
    for s in stages:
        vs.append(dict(kernel="splitk", smem_stages=s, prefetch="off"))
        for d in dists:
            vs.append(dict(kernel="splitk", smem_stages=s, prefetch="bulk", prefetch_distance=d))
        vs.append(dict(kernel="splitk", smem_stages=s, prefetch="line", prefetch_distance=4))
    for st in (8, 4, 12):
        vs.append(dict(kernel="balanced", smem_stages=st, prefetch="off"))
        vs.append(dict(kernel="balanced", smem_stages=st, prefetch="line", prefetch_distance=4))
        vs.append(dict(kernel="balanced", smem_stages=st, prefetch="bulk", prefetch_distance=4))
    for st, w in ((6, 2), (8, 1), (4, 2), (4, 4)):
        vs.append(dict(kernel="stream", smem_stages=st, stream_warps=w, prefetch="off"))
        vs.append(dict(kernel="stream", smem_stages=st, stream_warps=w, prefetch="line", prefetch_distance=4))
        if not quick:
            vs.append(dict(kernel="stream", smem_stages=st, stream_warps=w, prefetch="bulk", prefetch_distance=4))
    vs.append(dict(kernel="paper", prefetch="off"))
    for d in ([4] if quick else [1, 2, 4, 8, 16]):
        vs.append(dict(kernel="paper", prefetch="bulk", prefetch_distance=d))
    vs.append(dict(kernel="paper", prefetch="line", prefetch_distance=4))
    # 16-bit split-K with the producer-warp refill (the alternative to self-issue)
    vs.append(dict(kernel="splitk", smem_stages=8, prefetch="off", issue_mode="producer"))
    vs.append(dict(kernel="splitk", smem_stages=8, prefetch="line", prefetch_distance=4, issue_mode="producer"))
    # e4m3 KV cache (NEXT f3): library default ring (12 single / 16 paired by size), then fixed depths
    vs.append(dict(kernel="splitk", prefetch="off", kv="e4m3"))
    for st in (8, 16):
        vs.append(dict(kernel="splitk", smem_stages=st, prefetch="off", kv="e4m3"))
        vs.append(dict(kernel="splitk", smem_stages=st, prefetch="line", prefetch_distance=4, kv="e4m3"))
    # eviction priority: demand evict_first / prefetch evict_last / both
    for ev in (1, 2, 3):
        vs.append(dict(kernel="paper", prefetch="bulk", prefetch_distance=4, eviction=ev))
        vs.append(dict(kernel="splitk", smem_stages=8, prefetch="line", prefetch_distance=4, eviction=ev))
        vs.append(dict(kernel="splitk", smem_stages=4, prefetch="line", prefetch_distance=4, eviction=ev))
    vs.append(dict(kernel="paper", prefetch="off", eviction=1))
    vs.append(dict(kernel="splitk", smem_stages=8, prefetch="off", eviction=1))
    return vs


def cells(quick):
    import synth
    out = [synth.C2_LLAMA2_7B, synth.C3_LLAMA3_8B]
    bs = [1, 16, 64, 256] if quick else [1, 4, 16, 64, 256]
    cs = [512, 4096, 32768]
    for b in bs:
        for c in cs:
            out.append(synth.sweep_cell(b, c, seed=b * 7 + c))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "sweep.jsonl"))
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--reps", type=int, default=7)
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--cells", default="", help="comma list of cell names to keep")
    ap.add_argument("--kernels", default="", help="comma list of kernels to keep")
    ap.add_argument("--no-graphs", action="store_true", help="time direct calls instead of CUDA-graph replays")
    a = ap.parse_args()

    import torch

    import paper_2504_06319_b200 as pda
    import synth
    from bench import L2Flush
    pda.lib()
    flush = L2Flush(torch)
    keep = set(filter(None, a.cells.split(",")))
    f = open(a.out, "a")
    for cfg in cells(a.quick):
        if keep and cfg.name not in keep:
            continue
        inp = synth.make_inputs(cfg, seed=5, device="cuda")
        inp8 = synth.quantize_kv_e4m3(inp)
        kvb = cfg.kv_bytes()
        total = kvb + cfg.other_bytes()
        vs = variants(a.quick)
        if a.kernels:
            ks = set(a.kernels.split(","))
            vs = [v for v in vs if v["kernel"] in ks]
        times = {i: [] for i in range(len(vs))}
        outs = {}
        # separate zeroed workspaces: the stream kernel's arrival tickets must start at 0
        wss = {"splitk": torch.zeros(1 << 30, dtype=torch.uint8, device="cuda"),
               "stream": torch.zeros(256 << 20, dtype=torch.uint8, device="cuda"),
               "balanced": torch.zeros(256 << 20, dtype=torch.uint8, device="cuda"), "paper": None}
        graphs = {}
        for rnd in range(a.rounds):
            for i, v in enumerate(vs):

                def run(v=v, i=i):
                    kw = {k: x for k, x in v.items() if k != "kv"}
                    src = inp
                    if v.get("kv") == "e4m3":
                        src = inp8
                        kw.update(k_scale=inp8["k_scale"], v_scale=inp8["v_scale"])
                    return pda.paged_decode_attention(src["q"], src["k_cache"], src["v_cache"],
                                                      src["block_tables"], src["context_lens"],
                                                      src["scale"], out=outs.get(i),
                                                      workspace=wss[v["kernel"]], **kw)
                if rnd == 0:
                    outs[i] = run()
                    if not a.no_graphs:
                        g = torch.cuda.CUDAGraph()
                        with torch.cuda.graph(g, capture_error_mode="relaxed"):
                            run()
                        graphs[i] = g
                spans = []
                for _ in range(a.reps):  # all reps queued, one sync: no host gaps inside a span
                    flush()
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record()
                    if a.no_graphs:
                        run()
                    else:
                        graphs[i].replay()
                    e1.record()
                    spans.append((e0, e1))
                torch.cuda.synchronize()
                times[i].extend(e0.elapsed_time(e1) * 1e3 for e0, e1 in spans)
        # bitwise invariance of prefetch within each kernel/stages family
        for i, v in enumerate(vs):
            base = next(j for j, w in enumerate(vs) if w["kernel"] == v["kernel"]
                        and w.get("smem_stages") == v.get("smem_stages")
                        and w.get("stream_warps") == v.get("stream_warps") and w["prefetch"] == "off"
                        and not w.get("eviction") and w.get("kv") == v.get("kv")
                        and w.get("issue_mode") == v.get("issue_mode"))
            us = statistics.median(times[i])
            tot_v = (kvb // 2 + cfg.other_bytes()) if v.get("kv") == "e4m3" else total
            rec = dict(cell=cfg.name, batch=cfg.num_seqs, ctx=max(cfg.context_lens),
                       q_heads=cfg.num_q_heads, kv_heads=cfg.num_kv_heads, dtype=cfg.dtype,
                       kv_bytes=kvb, **v, us_median=us, us_p10=sorted(times[i])[len(times[i]) // 10],
                       us_p90=sorted(times[i])[(9 * len(times[i])) // 10], gbs=tot_v / (us * 1e-6) / 1e9,
                       speedup_vs_off=statistics.median(times[base]) / us,
                       bitwise_equal_to_off=bool(torch.equal(outs[i], outs[base])),
                       timing="cuda_graph_replay" if not a.no_graphs else "direct_call")
            f.write(json.dumps(rec) + "\n")
            f.flush()
            print(json.dumps(rec), flush=True)
        del inp, inp8, wss, outs, graphs
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
