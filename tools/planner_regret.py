"""(--small: partition-count sweep of small grids, see below.)  Planner regret scan: for each shape, the library default against a set of
alternative plans (partition size x2 / /2, merge forced, ring depth, the
tcgen05 kernel), timed interleaved with CUDA-graph replays after a clean L2
flush.  One JSON line per shape: default us, best alternative, regret =
default / best.  Cells where an alternative wins by more than a timer tick
point at planner rules to revisit.

    python tools/planner_regret.py [--out gpurun_out/regret.jsonl] [--rounds 5]
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2504_06319_b200 as pda
import synth
from bench import L2Flush

HEADS = [(32, 32), (32, 8), (64, 8), (8, 1), (4, 4), (32, 2)]
BATCH = [1, 8, 32, 128, 512]
CTX = [1024, 4096, 8192, 32768]
# --small: latency-bound grids (few (seq, kv head) rows), partition counts 1..64 x both merges
SMALL_HEADS = [(8, 1), (32, 8), (32, 32), (4, 4)]
SMALL_BATCH = [1, 2, 4, 8]
SMALL_CTX = [2048, 4096, 8192, 16384, 32768]


def small_variants(ctx):
    out = []
    for pm in (1, 2, 4, 8, 16, 32, 64):
        P = -(-ctx // pm)
        P = -(-P // 16) * 16
        if P < 128:
            continue
        if pm == 1:
            out.append(dict(partition_tokens=P))
        elif pm <= 8:
            out += [dict(partition_tokens=P, merge="combine"), dict(partition_tokens=P, merge="cluster")]
        else:
            out.append(dict(partition_tokens=P, merge="combine"))
    return out


def alternatives(plan):
    P = plan["partition_tokens"]
    alts = [dict(partition_tokens=P * 2), dict(smem_stages=12), dict(smem_stages=4)]
    if P >= 256:
        alts.append(dict(partition_tokens=P // 2))
    if plan["p_max"] > 1:
        alts += [dict(merge="combine"), dict(merge="cluster")] if plan["p_max"] <= 8 else [dict(merge="combine")]
    alts.append(dict(kernel="tc"))
    return alts


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/regret.jsonl")
    ap.add_argument("--rounds", type=int, default=5)
    ap.add_argument("--max-gb", type=float, default=4.5)
    ap.add_argument("--cells", default=None, help="comma-separated B_Hq_Hkv_ctx filter")
    ap.add_argument("--check", action="store_true", help="synchronize after every first replay (debug)")
    ap.add_argument("--small", action="store_true", help="partition-count sweep of small grids")
    ap.add_argument("--c4", action="store_true", help="ragged batch x context cells (BASELINE configs[3])")
    a = ap.parse_args()
    only = set(a.cells.split(",")) if a.cells else None
    flush = L2Flush(torch)
    ws = torch.zeros(1 << 30, dtype=torch.uint8, device="cuda")
    f = open(a.out, "w")
    heads, batch, ctxs = (SMALL_HEADS, SMALL_BATCH, SMALL_CTX) if a.small else (HEADS, BATCH, CTX)
    if a.c4:
        heads, batch, ctxs = [(32, 8)], [1, 4, 16, 32, 64, 128, 256], [512, 2048, 4096, 8192, 16384, 32768]
    for hq, hkv in heads:
        for B in batch:
            for ctx in ctxs:
                kv = 2 * B * hkv * ctx * 128 * 2
                if kv > a.max_gb * 1e9 or kv < 2e6:
                    continue
                if only and f"{B}_{hq}_{hkv}_{ctx}" not in only:
                    continue
                cfg = (synth.sweep_cell(B, ctx) if a.c4 else
                       synth.uniform(f"u_{B}_{hq}_{hkv}_128_{ctx}_bf16", B, hq, hkv, 128, ctx, "bf16"))
                kv = cfg.kv_bytes()
                if kv > a.max_gb * 1e9:
                    continue
                inp = synth.make_inputs(cfg, seed=0, device="cuda", poison=False)
                args = (inp["q"], inp["k_cache"], inp["v_cache"], inp["block_tables"], inp["context_lens"],
                        inp["scale"])
                out0 = pda.paged_decode_attention(*args, workspace=ws)
                plan = pda.plan(pda.make_shape(inp["q"], inp["k_cache"], inp["block_tables"]), pda.make_options())
                plan = {k: plan[k] for k in ("kernel", "p_max", "partition_tokens", "smem_stages", "cluster",
                                             "threads") if k in plan}
                variants = [dict()] + (small_variants(ctx) if a.small else alternatives(plan))
                graphs = []
                for v in variants:
                    try:
                        out = pda.paged_decode_attention(*args, workspace=ws, **v)
                        g = torch.cuda.CUDAGraph()
                        with torch.cuda.graph(g, capture_error_mode="relaxed"):
                            pda.paged_decode_attention(*args, out=out, workspace=ws, **v)
                        graphs.append((v, g, out))  # out stays alive as long as its graph (it writes there)
                        if a.check:
                            g.replay()
                            torch.cuda.synchronize()
                            print("ok", cfg.name, v, file=sys.stderr, flush=True)
                    except Exception as e:  # an alternative the planner refuses (unsupported)
                        print(json.dumps(dict(cell=cfg.name, variant=v, error=str(e)[:80])), file=sys.stderr)
                res = {i: [] for i in range(len(graphs))}
                for _ in range(a.rounds):
                    for i, (v, g, _) in enumerate(graphs):
                        spans = []
                        for rep in range(3):
                            flush()
                            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                            e0.record(); g.replay(); e1.record()
                            spans.append((e0, e1))
                            if a.check:
                                print("replay", cfg.name, v, rep, file=sys.stderr, flush=True)
                                torch.cuda.synchronize()
                        torch.cuda.synchronize()
                        res[i].extend(e0.elapsed_time(e1) * 1e3 for e0, e1 in spans)
                med = [statistics.median(res[i]) for i in range(len(graphs))]
                best = min(range(len(graphs)), key=lambda i: med[i])
                line = dict(cell=cfg.name, kv_gb=round(kv / 1e9, 3), plan=plan, default_us=round(med[0], 2),
                            best=graphs[best][0], best_us=round(med[best], 2), regret=round(med[0] / med[best], 3),
                            all={json.dumps(graphs[i][0]): round(med[i], 2) for i in range(len(graphs))})
                f.write(json.dumps(line) + "\n")
                f.flush()
                del inp, graphs, out0
                torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
