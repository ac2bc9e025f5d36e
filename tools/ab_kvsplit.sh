# split K / V ring (K slabs refilled right after QK^T; in-tree, PDA_KV_SPLIT=1) vs one barrier per
# stage refilled after PV (build_ab/nokvs, PDA_KV_SPLIT=0); library defaults, interleaved
N=build_ab/nokvs/libpda.so
for r in 1 2 3; do
  for c in c2 c3 c4_b64_ctx4096 c4_b256_ctx4096 u_128_8_1_128_8192_bf16 u_64_4_4_128_4096_fp16 c4_b4_ctx4096 c4_b1_ctx32768; do
    timeout 200 python tools/psweep.py $c '[dict()]' | sed 's/^/{"lib": "kvs", "r": '$r'} /'
    PDA_LIB_PATH=$N timeout 200 python tools/psweep.py $c '[dict()]' | sed 's/^/{"lib": "base", "r": '$r'} /'
  done
  for c in c2 c3 c4_b64_ctx4096 c4_b256_ctx4096 c4_b1_ctx32768; do
    timeout 200 python tools/psweep.py $c '[dict()]' kv8 | sed 's/^/{"lib": "kvs", "r": '$r'} /'
    PDA_LIB_PATH=$N timeout 200 python tools/psweep.py $c '[dict()]' kv8 | sed 's/^/{"lib": "base", "r": '$r'} /'
  done
done
timeout 120 python tools/l2res.py c2 '[dict()]' kv8 | sed 's/^/{"lib": "kvs"} /'
PDA_LIB_PATH=$N timeout 120 python tools/l2res.py c2 '[dict()]' kv8 | sed 's/^/{"lib": "base"} /'
