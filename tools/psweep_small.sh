# partition-size sweep on latency-bound cells (graph replays, L2 flushed)
V='[dict(), dict(partition_tokens=256), dict(partition_tokens=128), dict(partition_tokens=64)]'
for c in c4_b1_ctx512 c4_b1_ctx4096 c4_b1_ctx32768 c4_b4_ctx512 c4_b4_ctx4096 c4_b4_ctx32768 c4_b16_ctx512 c4_b16_ctx4096 c4_b64_ctx512; do
  python tools/psweep.py $c "$V"
done
