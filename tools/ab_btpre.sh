# (1) block ids loaded at CTA entry beside the length (in-tree) vs after it (build_ab/head)
# (2) software-pipelined consumers with a 12-stage ring (build_ab/swp, PDA_SWP=1) on the one-wave cells
H=build_ab/head/libpda.so; W=build_ab/swp/libpda.so
for r in 1 2 3; do
  for c in u_128_8_1_128_8192_bf16 u_128_32_2_128_8192_bf16 u_64_4_4_128_4096_fp16 c4_b16_ctx4096 c4_b64_ctx4096 c2 c4_b1_ctx4096; do
    timeout 200 python tools/psweep.py $c '[dict()]' | sed 's/^/{"lib": "btpre", "r": '$r'} /'
    PDA_LIB_PATH=$H timeout 200 python tools/psweep.py $c '[dict()]' | sed 's/^/{"lib": "head", "r": '$r'} /'
  done
  for c in u_128_8_1_128_8192_bf16 u_128_32_2_128_8192_bf16 u_64_4_4_128_4096_fp16; do
    PDA_LIB_PATH=$W timeout 200 python tools/psweep.py $c '[dict(), dict(smem_stages=12)]' | sed 's/^/{"lib": "swp", "r": '$r'} /'
    PDA_LIB_PATH=$H timeout 200 python tools/psweep.py $c '[dict(smem_stages=12)]' | sed 's/^/{"lib": "head", "r": '$r'} /'
  done
done
