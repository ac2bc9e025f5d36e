# warp-uniform indices (lane-0 shuffle) + elect.sync refill issue from the converged warp (in-tree: no
# per-load ELECT / R2UR.BROADCAST loop in the SASS) vs the lane == 0 issue (build_ab/head2); interleaved
H=build_ab/head2/libpda.so
for r in 1 2 3; do
  for c in c2 c3 c4_b64_ctx4096 u_128_8_1_128_8192_bf16 u_128_32_2_128_8192_bf16 u_64_4_4_128_4096_fp16 c4_b16_ctx4096 c4_b1_ctx32768; do
    timeout 200 python tools/psweep.py $c '[dict()]' | sed 's/^/{"lib": "new", "r": '$r'} /'
    PDA_LIB_PATH=$H timeout 200 python tools/psweep.py $c '[dict()]' | sed 's/^/{"lib": "head", "r": '$r'} /'
  done
  for c in c2 c3 c4_b64_ctx4096 c4_b256_ctx4096 c4_b1_ctx32768; do
    timeout 200 python tools/psweep.py $c '[dict()]' kv8 | sed 's/^/{"lib": "new", "r": '$r'} /'
    PDA_LIB_PATH=$H timeout 200 python tools/psweep.py $c '[dict()]' kv8 | sed 's/^/{"lib": "head", "r": '$r'} /'
  done
done
for c in c2 u_128_8_1_128_8192_bf16; do
  timeout 120 python tools/l2res.py $c '[dict()]' | sed 's/^/{"lib": "new"} /'
  PDA_LIB_PATH=$H timeout 120 python tools/l2res.py $c '[dict()]' | sed 's/^/{"lib": "head"} /'
done
timeout 120 python tools/l2res.py c2 '[dict()]' kv8 | sed 's/^/{"lib": "new"} /'
PDA_LIB_PATH=$H timeout 120 python tools/l2res.py c2 '[dict()]' kv8 | sed 's/^/{"lib": "head"} /'
