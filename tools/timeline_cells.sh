# per-CTA timelines of the default plan on the bench and sweep cells
for c in c4_b64_ctx4096 c4_b16_ctx4096 c4_b256_ctx512 c4_b256_ctx4096 c4_b16_ctx32768 c2 c3; do
  python tools/timeline.py $c
done
python tools/timeline.py c4_b64_ctx4096 "dict(partition_tokens=2048)"
python tools/timeline.py c4_b64_ctx4096 "dict(partition_tokens=512)"
python tools/timeline.py c2 "{}" kv8
