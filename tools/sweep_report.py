"""Markdown report of a tools/sweep.py JSONL (profiles/).

    python tools/sweep_report.py profiles/r01_sweep_final.jsonl > profiles/r01_sweep_final.md
"""
import json
import sys


def main():
    path = sys.argv[1]
    rows = [json.loads(l) for l in open(path)]
    assert all(r["bitwise_equal_to_off"] for r in rows), "a prefetch/eviction variant changed a result"
    cells = list(dict.fromkeys(r["cell"] for r in rows))

    def get(c, **kw):
        out = [r for r in rows if r["cell"] == c and all(r.get(k) == v for k, v in kw.items())]
        for k in ("eviction", "issue_mode", "kv"):
            if k not in kw:
                out = [r for r in out if not r.get(k)]
        return out[0] if out else None

    def name(r):
        s = r["kernel"]
        if r.get("smem_stages"):
            s += f" S{r['smem_stages']}"
        if r.get("stream_warps"):
            s += f"w{r['stream_warps']}"
        s += " " + r["prefetch"] + (f" d{r['prefetch_distance']}" if r["prefetch"] != "off" else "")
        for k in ("eviction", "issue_mode", "kv"):
            if r.get(k):
                s += f" {k}={r[k]}"
        return s

    x = lambda r: f"{r['speedup_vs_off']:.3f}" if r else "-"
    us = lambda r: f"{r['us_median']:.1f}" if r else "-"
    print(f"# Sweep report ({path.split('/')[-1]})\n")
    print("One B200; per cell all variants on the same inputs, interleaved rounds of graph replays, an L2 "
          "flush before each iteration (512 MiB write + 256 MiB read in the newer sweeps, write only in the "
          "older ones, which then charge the step up to 126 MB of dirty-line write-back), CUDA-event median of a CUDA-graph replay.  Every prefetch / eviction "
          f"variant's output is bitwise equal to the same kernel with prefetch off ({len(rows)} lines, asserted). "
          "GB/s = algorithmic bytes (KV + q + out + block tables; e4m3 KV counts 1 B/element) / time.\n")
    print("## Kernels\n")
    print("| cell | B | ctx | KV GB | library default µs | GB/s | split-K self-issue S8 µs | split-K producer-warp µs | "
          "best split-K variant | balanced best µs | stream best µs | paper kernel µs | e4m3 KV µs (library default; S16 in older sweeps) | "
          "e4m3 speedup |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|---|---|")
    for c in cells:
        rs = [r for r in rows if r["cell"] == c]
        d8 = get(c, kernel="splitk", smem_stages=8, prefetch="off")
        d = get(c, kernel="splitk", smem_stages=None, prefetch="off") or d8
        pr = get(c, kernel="splitk", smem_stages=8, prefetch="off", issue_mode="producer")
        sk = min([r for r in rs if r["kernel"] == "splitk" and not r.get("kv")], key=lambda r: r["us_median"])
        bal = min([r for r in rs if r["kernel"] == "balanced"], key=lambda r: r["us_median"])
        st = min([r for r in rs if r["kernel"] == "stream"], key=lambda r: r["us_median"])
        pp = get(c, kernel="paper", prefetch="off")
        e8 = (get(c, kernel="splitk", smem_stages=None, prefetch="off", kv="e4m3")
              or get(c, kernel="splitk", smem_stages=16, prefetch="off", kv="e4m3"))
        print(f"| {c} | {d['batch']} | {d['ctx']} | {d['kv_bytes'] / 1e9:.3f} | {us(d)} | {d['gbs']:.0f} | {us(d8)} | "
              f"{us(pr)} | {name(sk)}: {us(sk)} | {us(bal)} | {us(st)} | {us(pp)} | {us(e8)} | "
              f"{(d['us_median'] / e8['us_median']) if e8 else 0:.2f}x |")
    print("\n## Prefetch and eviction priority (speedup vs the same configuration with prefetch off)\n")
    print("| cell | paper kernel: bulk d4 (Alg. 1) | line d4 | bulk d4 + prefetch evict_last | split-K self S8: line d4 | "
          "bulk d4 | bulk d16 | split-K S4: line d4 | split-K producer S8: line d4 | e4m3 S8: line d4 | "
          "split-K S8 demand evict_first (no prefetch) |")
    print("|---|---|---|---|---|---|---|---|---|---|---|")
    for c in cells:
        ev1 = get(c, kernel="splitk", smem_stages=8, prefetch="off", eviction=1)
        base = get(c, kernel="splitk", smem_stages=8, prefetch="off")
        ev1s = f"{base['us_median'] / ev1['us_median']:.3f}" if ev1 else "-"
        print(f"| {c} | {x(get(c, kernel='paper', prefetch='bulk', prefetch_distance=4))} | "
              f"{x(get(c, kernel='paper', prefetch='line'))} | "
              f"{x(get(c, kernel='paper', prefetch='bulk', prefetch_distance=4, eviction=2))} | "
              f"{x(get(c, kernel='splitk', smem_stages=8, prefetch='line'))} | "
              f"{x(get(c, kernel='splitk', smem_stages=8, prefetch='bulk', prefetch_distance=4))} | "
              f"{x(get(c, kernel='splitk', smem_stages=8, prefetch='bulk', prefetch_distance=16))} | "
              f"{x(get(c, kernel='splitk', smem_stages=4, prefetch='line'))} | "
              f"{x(get(c, kernel='splitk', smem_stages=8, prefetch='line', issue_mode='producer'))} | "
              f"{x(get(c, kernel='splitk', smem_stages=8, prefetch='line', kv='e4m3'))} | {ev1s} |")


if __name__ == "__main__":
    main()
