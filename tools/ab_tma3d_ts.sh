# 3-D vs 2-D TMA boxes with the round-2 default planner (split kernel on one-wave cells), 3 interleaved rounds
A=build_ab/tma2d/libpda.so
for r in 1 2 3; do
  for c in u_128_32_2_128_8192_bf16 u_128_8_1_128_8192_bf16 c4_b64_ctx4096 u_64_4_4_128_4096_fp16 c2; do
    timeout 120 python tools/l2res.py $c | sed 's/^/{"lib": "3d", "r": '$r'} /'
    PDA_LIB_PATH=$A timeout 120 python tools/l2res.py $c | sed 's/^/{"lib": "2d", "r": '$r'} /'
  done
done
