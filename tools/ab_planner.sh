# planner A/B in one run: default (NEW) vs PDA_PLANNER_V1=1 (OLD), interleaved
for r in 1 2; do
for c in c4_b4_ctx32768 c4_b16_ctx4096 c4_b16_ctx32768 u_24_32_8_128_4096_bf16 u_32_32_8_128_8192_bf16 u_64_4_4_128_4096_fp16 u_256_8_1_128_16384_bf16 c4_b64_ctx4096; do
  echo "NEW $c $(python tools/psweep.py $c '[dict()]' | tail -1)"
  echo "OLD $c $(PDA_PLANNER_V1=1 python tools/psweep.py $c '[dict()]' | tail -1)"
done; done
