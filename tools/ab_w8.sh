# A/B: 8 consumer warps (auto rule: one wave at 2 CTAs/SM) vs forced 4
for r in 1 2; do
  for c in u_1_32_32_128_32768_bf16 u_8_16_16_128_8192_bf16 u_32_28_4_128_8192_bf16 u_8_32_8_128_8192_bf16 c4_b16_ctx4096 c4_b4_ctx32768 c4_b1_ctx32768 c4_b16_ctx512 u_1_8_1_128_32768_bf16 c1; do
    echo "W8 $c $(python tools/psweep.py $c '[dict()]' | tail -1)"
    echo "W4 $c $(PDA_SPLITK_WARPS=4 python tools/psweep.py $c '[dict()]' | tail -1)"
  done
done
