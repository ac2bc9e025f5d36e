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
    dict(kernel="splitk", smem_stages=4, prefetch="off"),
    dict(kernel="splitk", smem_stages=4, prefetch="line", prefetch_distance=4),
    dict(kernel="splitk", smem_stages=8, prefetch="off"),
    dict(kernel="splitk", smem_stages=8, prefetch="bulk", prefetch_distance=4),
    dict(kernel="splitk", smem_stages=8, prefetch="line", prefetch_distance=4),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    a = ap.parse_args()
    import torch

    import paper_2504_06319_b200 as pda
    import synth
    sys.path.insert(0, ROOT)
    from bench import workload_config
    cfg = workload_config(a.config)
    inp = synth.make_inputs(cfg, seed=5, device="cuda")
    ws = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
    order = []
    for v in VARIANTS:
        for rep in range(2):
            pda.paged_decode_attention(inp["q"], inp["k_cache"], inp["v_cache"], inp["block_tables"],
                                       inp["context_lens"], inp["scale"], workspace=ws, **v)
            order.append(dict(v, rep=rep))
    torch.cuda.synchronize()
    with open(os.path.join(ROOT, "gpurun_out", f"ablation_order_{a.config}.json"), "w") as f:
        json.dump(order, f)
    print(json.dumps(order))


if __name__ == "__main__":
    main()
