# tc kernel variants: default (128-token tiles x 3 stages, K as one 4-D box per block, lane-parallel
# TMA issue) vs lane-0 issue vs 64-token tiles x 6 stages vs K as two 2-D boxes per block
for lib in default build_ab/tc_nopar/libpda.so build_ab/tc_m64/libpda.so build_ab/tc_k2d/libpda.so; do
  for c in c2 u_128_8_1_128_8192_bf16 c4_b64_ctx4096; do
    if [ $lib = default ]; then python tools/l2res.py $c '[dict(kernel="tc")]'; else PDA_LIB_PATH=$lib python tools/l2res.py $c '[dict(kernel="tc")]'; fi | sed "s#^#{\"lib\": \"$lib\"} #"
  done
done
python tools/tc_check.py parity
