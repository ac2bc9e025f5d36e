"""Per-CTA timeline of one split-K decode step (paged_decode_attention_timeline).

    python tools/timeline.py c4_b64_ctx4096 ["dict(partition_tokens=2048)"] [kv8]

Each unit CTA records %globaltimer at entry and exit and its SM.  From those
and the trace's visited-block counts this prints: the kernel span, the
number of resident CTAs over time (1 us bins, summarised), the bytes each
CTA streamed / its lifetime, the ramp (first entry -> 90 % of peak
residency) and the drain (residency falling below 50 % of peak -> last
exit), and an estimate of the bandwidth lost to the drain.  The trace
instantiation runs a few percent slower than the product kernel; the
shares, not the absolute times, are the point.  One JSON line on stdout.
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2504_06319_b200 as pda
import synth
from bench import L2Flush, workload_config


def main():
    cfg = workload_config(sys.argv[1])
    kw = eval(sys.argv[2]) if len(sys.argv) > 2 else {}
    kv8 = len(sys.argv) > 3 and sys.argv[3] == "kv8"
    inp = synth.make_inputs(cfg, seed=0, device="cuda")
    if kv8:
        inp = synth.quantize_kv_e4m3(inp)
        kw.update(k_scale=inp["k_scale"], v_scale=inp["v_scale"])
    args = (inp["q"], inp["k_cache"], inp["v_cache"], inp["block_tables"], inp["context_lens"], inp["scale"])
    flush = L2Flush(torch)
    for _ in range(3):
        pda.paged_decode_attention(*args, **kw)
    # plain product step time (events, flushed) for reference
    times = []
    for _ in range(5):
        flush()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        pda.paged_decode_attention(*args, **kw)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) * 1e3)
    best = None
    for _ in range(3):
        flush()
        out, tr, info, st = pda.paged_decode_attention(*args, timeline=True, **kw)
        torch.cuda.synchronize()
        span = int(st[:, 1].max() - st[:, 0][st[:, 0] > 0].min())
        if best is None or span < best[0]:
            best = (span, tr.cpu(), info, st.cpu())
    _, tr, info, st = best
    rec = tr.view(info["trace_records"], info["trace_rec_len"])
    nblk = rec[:, 2].clamp(min=0).to(torch.int64)
    elem = 1 if kv8 else 2
    blk_bytes = 2 * 16 * cfg.head_dim * elem  # K + V slab of one (block, kv head)
    live = st[:, 0] > 0
    t0 = int(st[live, 0].min())
    s = (st[live, 0] - t0).double() / 1e3  # us
    e = (st[live, 1] - t0).double() / 1e3
    b = (nblk[live] * blk_bytes).double()
    work = b > 0
    T = float(e.max())
    # residency (CTAs alive) and streamed bytes per 1 us bin (bytes spread evenly over a CTA's life)
    nb = int(T) + 1
    res = torch.zeros(nb, dtype=torch.float64)
    bw = torch.zeros(nb, dtype=torch.float64)
    for si, ei, bi in zip(s.tolist(), e.tolist(), b.tolist()):
        lo, hi = int(si), min(int(ei), nb - 1)
        dur = max(ei - si, 1e-3)
        for k in range(lo, hi + 1):
            ov = min(ei, k + 1) - max(si, k)
            if ov > 0:
                res[k] += ov
                bw[k] += bi * ov / dur
    peak_res = float(res.max())
    ramp_end = next(k for k in range(nb) if res[k] >= 0.9 * peak_res)
    drain_start = max(k for k in range(nb) if res[k] >= 0.5 * peak_res)
    body = bw[ramp_end:drain_start]
    body_rate = float(body.mean()) if len(body) else float(bw.mean())  # bytes per us in the steady state
    total = float(b.sum())
    ideal = total / body_rate if body_rate > 0 else T
    life = (e - s)[work]
    rate = (b[work] / (e - s)[work]) / 1e3  # GB/s per CTA
    # per-SM load: how many CTAs ran on the SM over the whole kernel (= CTAs sharing it in a
    # one-wave grid) vs the rate each streamed
    sm = st[live, 2][work].tolist()
    from collections import Counter, defaultdict
    per_sm = Counter(sm)
    by_load = defaultdict(list)
    for smi, r in zip(sm, rate.tolist()):
        by_load[per_sm[smi]].append(r)
    sm_rates = {f"{k}_ctas_on_sm": dict(n_ctas=len(v), gbs_per_cta=round(statistics.median(v), 2))
                for k, v in sorted(by_load.items())}
    line = dict(cell=cfg.name + ("_kv8" if kv8 else ""), **{k: v for k, v in kw.items() if not k.endswith("scale")},
                plan=dict(p_max=info["p_max"], partition_tokens=info["partition_tokens"], cluster=info["cluster"],
                          grid=[info["grid_x"], info["grid_y"], info["grid_z"]]),
                step_us_events=round(statistics.median(times), 1), trace_kernel_span_us=round(T, 1),
                units=int(live.sum()), units_with_work=int(work.sum()), bytes=int(total),
                peak_resident=round(peak_res, 1), ramp_us=ramp_end, drain_us=round(T - drain_start, 1),
                steady_gbs=round(body_rate / 1e3, 1), span_at_steady_rate_us=round(ideal, 1),
                lost_to_ramp_and_drain_us=round(T - ideal, 1),
                cta_life_us=dict(p10=round(float(life.quantile(0.1)), 1), p50=round(float(life.median()), 1),
                                 p90=round(float(life.quantile(0.9)), 1)),
                cta_gbs=dict(p10=round(float(rate.quantile(0.1)), 2), p50=round(float(rate.median()), 2),
                             p90=round(float(rate.quantile(0.9)), 2)),
                sms_used=int(st[live, 2].unique().numel()), per_sm_load=sm_rates,
                residency_1us=[round(float(x), 1) for x in res[:: max(1, nb // 40)]],
                gbs_1us=[round(float(x) / 1e3) for x in bw[:: max(1, nb // 40)]])
    print(json.dumps(line))


if __name__ == "__main__":
    main()
