"""Summarise a tools/sweep.py JSONL into a markdown table (profiles/).

    python tools/sweep_table.py profiles/r01_sweep.jsonl > profiles/r01_sweep.md
"""
import json
import sys
from collections import OrderedDict


def main():
    rows = [json.loads(l) for l in open(sys.argv[1])]
    assert all(r["bitwise_equal_to_off"] for r in rows), "prefetch changed a result"
    cells = OrderedDict()
    for r in rows:
        cells.setdefault(r["cell"], []).append(r)
    print("| cell | B | ctx | KV GB | splitk S8 off µs | GB/s | S8 line d4 | S4 off µs | S4 best prefetch | "
          "S8 bulk d4 | S8 bulk d16 | paper off µs | GB/s | paper bulk d4 (Alg. 1) | paper line d4 | paper best |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|")
    for c, rs in cells.items():
        def get(**kw):
            return [r for r in rs if all(r.get(k) == v for k, v in kw.items())]
        s8 = get(kernel="splitk", smem_stages=8, prefetch="off")[0]
        s8l = get(kernel="splitk", smem_stages=8, prefetch="line")[0]
        s4 = get(kernel="splitk", smem_stages=4, prefetch="off")[0]
        s4b = max(get(kernel="splitk", smem_stages=4), key=lambda r: r["speedup_vs_off"])
        s8b4 = get(kernel="splitk", smem_stages=8, prefetch="bulk", prefetch_distance=4)[0]
        s8b16 = get(kernel="splitk", smem_stages=8, prefetch="bulk", prefetch_distance=16)
        po = get(kernel="paper", prefetch="off")[0]
        pb = get(kernel="paper", prefetch="bulk", prefetch_distance=4)[0]
        pl = get(kernel="paper", prefetch="line")[0]
        pbest = max(get(kernel="paper"), key=lambda r: r["speedup_vs_off"])
        name = lambda r: r["prefetch"] + (f" d{r['prefetch_distance']}" if r["prefetch"] != "off" else "")
        print(f"| {c} | {s8['batch']} | {s8['ctx']} | {s8['kv_bytes'] / 1e9:.3f} | {s8['us_median']:.1f} | "
              f"{s8['gbs']:.0f} | x{s8l['speedup_vs_off']:.3f} | {s4['us_median']:.1f} | "
              f"{name(s4b)} x{s4b['speedup_vs_off']:.3f} | x{s8b4['speedup_vs_off']:.3f} | "
              f"{('x%.3f' % s8b16[0]['speedup_vs_off']) if s8b16 else '-'} | {po['us_median']:.1f} | "
              f"{po['gbs']:.0f} | x{pb['speedup_vs_off']:.3f} | x{pl['speedup_vs_off']:.3f} | "
              f"{name(pbest)} x{pbest['speedup_vs_off']:.3f} |")


if __name__ == "__main__":
    main()
