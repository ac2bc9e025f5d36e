# e4m3 small grids under the small-grid planner (<= 256 CTAs) vs round-2 HEAD (build_ab/head)
H=build_ab/head/libpda.so
for r in 1 2 3; do
  for c in c4_b1_ctx4096 c4_b1_ctx32768 c4_b2_ctx32768 u_1_8_1_128_8192_bf16 u_1_8_1_128_32768_bf16 u_2_32_8_128_8192_bf16 u_4_4_4_128_32768_bf16 u_1_32_32_128_8192_bf16 u_8_8_1_128_16384_bf16; do
    timeout 200 python tools/psweep.py $c '[dict()]' kv8 | sed 's/^/{"lib": "new", "r": '$r'} /'
    PDA_LIB_PATH=$H timeout 200 python tools/psweep.py $c '[dict()]' kv8 | sed 's/^/{"lib": "head", "r": '$r'} /'
  done
done
