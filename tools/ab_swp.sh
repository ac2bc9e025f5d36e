# software-pipelined consumers (QK^T of the next block before this one's softmax/PV; PDA_SWP=1,
# the in-tree build) vs one chain at a time (build_ab/noswp, -DPDA_SWP=0), interleaved, graph
# replays: HBM (L2 flushed) and L2-resident timings per cell (tools/l2res.py)
A=build_ab/noswp/libpda.so
for r in 1 2 3; do
  for c in u_128_8_1_128_8192_bf16 u_128_32_2_128_8192_bf16 c4_b64_ctx4096 c4_b16_ctx4096 c2 c3; do
    timeout 120 python tools/l2res.py $c | sed 's/^/{"lib": "swp", "r": '$r'} /'
    PDA_LIB_PATH=$A timeout 120 python tools/l2res.py $c | sed 's/^/{"lib": "noswp", "r": '$r'} /'
  done
  for c in c2 c3 c4_b64_ctx4096; do
    timeout 120 python tools/l2res.py $c '[dict()]' kv8 | sed 's/^/{"lib": "swp", "kv8": 1, "r": '$r'} /'
    PDA_LIB_PATH=$A timeout 120 python tools/l2res.py $c '[dict()]' kv8 | sed 's/^/{"lib": "noswp", "kv8": 1, "r": '$r'} /'
  done
done
