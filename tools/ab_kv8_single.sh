# e4m3: 16-stage ring consumed in pairs (default) vs one block at a time (build_ab/kv8single,
# PDA_KV8_PAIRS=0: a warp holds one of its four stages, not two) vs that plus the software pipeline
# (build_ab/kv8single_swp, PDA_SWP=1); library defaults otherwise, interleaved
S=build_ab/kv8single/libpda.so; W=build_ab/kv8single_swp/libpda.so
for r in 1 2 3; do
  for c in c2 c3 c4_b256_ctx4096 c4_b64_ctx8192 u_128_8_1_128_8192_bf16; do
    timeout 200 python tools/psweep.py $c '[dict(smem_stages=16)]' kv8 | sed 's/^/{"lib": "pairs", "r": '$r'} /'
    PDA_LIB_PATH=$S timeout 200 python tools/psweep.py $c '[dict(smem_stages=16)]' kv8 | sed 's/^/{"lib": "single", "r": '$r'} /'
    PDA_LIB_PATH=$W timeout 200 python tools/psweep.py $c '[dict(smem_stages=16)]' kv8 | sed 's/^/{"lib": "single_swp", "r": '$r'} /'
  done
done
for L in pairs single single_swp; do
  P=; [ $L = single ] && P=$S; [ $L = single_swp ] && P=$W
  PDA_LIB_PATH=$P timeout 120 python tools/l2res.py c2 '[dict(smem_stages=16)]' kv8 | sed 's/^/{"lib": "'$L'"} /'
done
