# S8 combine kernel: every load issued up front (in-tree) vs the dependent lens -> lse -> o chain (build_ab/oldcomb)
A=build_ab/oldcomb/libpda.so
for r in 1 2 3; do
  for c in c4_b64_ctx4096 c4_b16_ctx4096 c4_b256_ctx4096 c4_b16_ctx32768 c4_b64_ctx32768 c3 u_74_8_1_128_16384_bf16 u_1_32_32_128_32768_bf16; do
    timeout 200 python tools/psweep.py $c '[dict()]' | sed 's/^/{"lib": "upfront", "r": '$r'} /'
    PDA_LIB_PATH=$A timeout 200 python tools/psweep.py $c '[dict()]' | sed 's/^/{"lib": "chain", "r": '$r'} /'
  done
done
