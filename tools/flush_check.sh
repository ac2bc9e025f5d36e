# clean flush (write + read) vs bench's unflushed back-to-back steps, and the mid cells
for c in c2 c3 c4_b64_ctx4096 c4_b256_ctx4096 c4_b16_ctx32768 c4_b64_ctx32768 c4_b16_ctx4096 c4_b256_ctx512; do
  python tools/psweep.py $c '[dict()]' | tail -1
done
