# CTA start-up: block ids beside the length + tensor-map prefetch and ring-barrier init at entry (in-tree)
# vs round-2 HEAD before them (build_ab/head); flushed single steps (psweep) and back to back
H=build_ab/head/libpda.so
for r in 1 2 3; do
  for c in u_128_8_1_128_8192_bf16 u_64_4_4_128_4096_fp16 c4_b16_ctx4096 c4_b1_ctx4096 c4_b64_ctx512 c1; do
    timeout 200 python tools/psweep.py $c '[dict()]' | sed 's/^/{"lib": "new", "r": '$r'} /'
    PDA_LIB_PATH=$H timeout 200 python tools/psweep.py $c '[dict()]' | sed 's/^/{"lib": "head", "r": '$r'} /'
  done
done
for r in 1 2; do
  timeout 300 python tools/backtoback.py u_128_8_1_128_8192_bf16 u_64_4_4_128_4096_fp16 c4_b16_ctx4096 c2 | sed 's/^/{"lib": "new", "r": '$r'} /'
  PDA_LIB_PATH=$H timeout 300 python tools/backtoback.py u_128_8_1_128_8192_bf16 u_64_4_4_128_4096_fp16 c4_b16_ctx4096 c2 | sed 's/^/{"lib": "head", "r": '$r'} /'
done
