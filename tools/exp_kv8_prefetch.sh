# e4m3 cache: the paper's L2 prefetch beyond the smem ring (line / bulk, distance d, evict_last on the prefetches)
V='[dict(prefetch="off"), dict(prefetch="line", prefetch_distance=4), dict(prefetch="line", prefetch_distance=8), dict(prefetch="line", prefetch_distance=16), dict(prefetch="bulk", prefetch_distance=4), dict(prefetch="bulk", prefetch_distance=8), dict(prefetch="bulk", prefetch_distance=16), dict(prefetch="line", prefetch_distance=8, eviction="both"), dict(prefetch="bulk", prefetch_distance=8, eviction="both")]'
for c in c2 c3 c4_b64_ctx4096 c4_b256_ctx4096; do
  timeout 300 python tools/psweep.py $c "$V" kv8
done
timeout 300 python tools/psweep.py c2 "$V"
