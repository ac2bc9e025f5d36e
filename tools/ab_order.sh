# partition-major grid order A/B (PDA_PART_MAJOR=1 vs 0), interleaved
for r in 1 2; do
for c in c4_b64_ctx4096 c4_b256_ctx4096 c4_b16_ctx32768 c4_b64_ctx32768 c4_b256_ctx512 c4_b64_ctx512 c3 c4_b256_ctx32768; do
  echo "PM1 $c $(PDA_PART_MAJOR=1 python tools/psweep.py $c '[dict()]' | tail -1)"
  echo "PM0 $c $(PDA_PART_MAJOR=0 python tools/psweep.py $c '[dict()]' | tail -1)"
done; done
