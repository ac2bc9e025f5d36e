"""One launch per prefetch-ablation variant, for ncu capture (paper Table 3 analog).

    ncu --set full -k regex:'paper_kernel|splitk_kernel' -o gpurun_out/ablation \
        python tools/ablation_launches.py --config c2

Each variant runs once untimed (module load / warm-up) and once for capture,
so with `-s` unset ncu captures both; the summary tool keeps the second.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

VARIANTS = [
    dict(kernel="paper", prefetch="off"),
    dict(kernel="paper", prefetch="bulk", prefetch_distance=4),
    dict(kernel="paper", prefetch="line", prefetch_distance=4),
    dict(kernel="splitk", smem_stages=8, prefetch="off", issue_mode="producer"),
    dict(kernel="splitk", smem_stages=8, prefetch="line", prefetch_distance=4, issue_mode="producer"),
    dict(kernel="splitk", smem_stages=8, prefetch="off"),
    dict(kernel="splitk", smem_stages=8, prefetch="bulk", prefetch_distance=4),
    dict(kernel="splitk", smem_stages=8, prefetch="line", prefetch_distance=4),
    dict(kernel="splitk", smem_stages=16, prefetch="off", kv="e4m3"),
    dict(kernel="splitk", smem_stages=8, prefetch="line", prefetch_distance=4, kv="e4m3"),
]


# the batch x context grid (BASELINE configs[3]): paper and
# split-K kernels, prefetch off / on, at the library's default ring and eviction
GRID_VARIANTS = [
    dict(kernel="paper", prefetch="off"),
    dict(kernel="paper", prefetch="bulk", prefetch_distance=4),
    dict(kernel="paper", prefetch="bulk", prefetch_distance=4, eviction="prefetch_last"),
    dict(kernel="paper", prefetch="line", prefetch_distance=4),
    dict(kernel="splitk", prefetch="off"),
    dict(kernel="splitk", prefetch="line", prefetch_distance=4),
    dict(kernel="splitk", prefetch="bulk", prefetch_distance=4),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--grid", action="store_true", help="the C4 grid variant list (GRID_VARIANTS)")
    a = ap.parse_args()
    variants = GRID_VARIANTS if a.grid else VARIANTS
    import torch

    import paper_2504_06319_b200 as pda
    import synth
    sys.path.insert(0, ROOT)
    from bench import workload_config
    cfg = workload_config(a.config)
    inp = synth.make_inputs(cfg, seed=5, device="cuda")
    inp8 = synth.quantize_kv_e4m3(inp) if any(v.get("kv") == "e4m3" for v in variants) else None
    ws = torch.zeros(1 << 30, dtype=torch.uint8, device="cuda")
    order = []
    for v in variants:
        kw = {k: x for k, x in v.items() if k != "kv"}
        src = inp
        if v.get("kv") == "e4m3":
            src = inp8
            kw.update(k_scale=inp8["k_scale"], v_scale=inp8["v_scale"])
        for rep in range(2):
            pda.paged_decode_attention(src["q"], src["k_cache"], src["v_cache"], src["block_tables"],
                                       src["context_lens"], src["scale"], workspace=ws, **kw)
            order.append(dict(v, rep=rep))
    torch.cuda.synchronize()
    with open(os.path.join(ROOT, "gpurun_out", f"ablation_order_{a.config}.json"), "w") as f:
        json.dump(order, f)
    print(json.dumps(order))


if __name__ == "__main__":
    main()
