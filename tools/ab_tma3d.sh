# one 3-D TMA box per 16-bit slab (default) vs two 2-D boxes (PDA_TMA3D=0 build)
A=build_ab/tma2d/libpda.so
for c in u_128_8_1_128_8192_bf16 u_128_32_2_128_8192_bf16 c4_b64_ctx4096 c4_b16_ctx4096 c2 c3; do
  for r in 1 2; do
    python tools/l2res.py $c | sed 's/^/{"lib": "3d", "r": '$r'} /'
    PDA_LIB_PATH=$A python tools/l2res.py $c | sed 's/^/{"lib": "2d", "r": '$r'} /'
  done
done
