# small-grid planner (<= 8 rows: <= 128 CTAs, partitions >= min(ctx/16, 1024); cluster merge only from
# one CTA per SM) in-tree vs round-2 HEAD before it (build_ab/head), library defaults, interleaved
H=build_ab/head/libpda.so
for r in 1 2 3; do
  for c in u_1_8_1_128_4096_bf16 u_1_8_1_128_8192_bf16 u_1_8_1_128_16384_bf16 u_1_8_1_128_32768_bf16 u_2_8_1_128_8192_bf16 u_4_8_1_128_32768_bf16 u_8_8_1_128_4096_bf16 u_1_32_8_128_2048_bf16 u_1_32_8_128_4096_bf16 u_1_32_8_128_32768_bf16 u_2_32_8_128_2048_bf16 u_4_4_4_128_2048_bf16 u_1_4_4_128_32768_bf16 u_2_4_4_128_8192_bf16 u_8_4_4_128_32768_bf16 u_1_32_32_128_1024_bf16 u_1_32_32_128_32768_bf16 c4_b1_ctx4096 c4_b1_ctx32768 c4_b4_ctx32768 c4_b16_ctx4096 c1 c4_b1_ctx512 c4_b4_ctx512; do
    timeout 200 python tools/psweep.py $c '[dict()]' | sed 's/^/{"lib": "new", "r": '$r'} /'
    PDA_LIB_PATH=$H timeout 200 python tools/psweep.py $c '[dict()]' | sed 's/^/{"lib": "head", "r": '$r'} /'
  done
  for c in c4_b1_ctx4096 c4_b1_ctx32768 c4_b4_ctx32768 u_1_8_1_128_8192_bf16; do
    timeout 200 python tools/psweep.py $c '[dict()]' kv8 | sed 's/^/{"lib": "new", "r": '$r'} /'
    PDA_LIB_PATH=$H timeout 200 python tools/psweep.py $c '[dict()]' kv8 | sed 's/^/{"lib": "head", "r": '$r'} /'
  done
done
