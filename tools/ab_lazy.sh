# lazy softmax reference (R24) vs the eager per-block rescale (build_ab/tc_base), interleaved
A=build_ab/tc_base/libpda.so
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "lazy or rescale" 2>&1 | tail -3
for r in 1 2 3; do
  for c in u_128_8_1_128_8192_bf16 u_128_32_2_128_8192_bf16 c4_b64_ctx4096 c4_b16_ctx4096 c2 c3; do
    timeout 120 python tools/l2res.py $c | sed 's/^/{"lib": "lazy", "r": '$r'} /'
    PDA_LIB_PATH=$A timeout 120 python tools/l2res.py $c | sed 's/^/{"lib": "eager", "r": '$r'} /'
  done
  timeout 120 python tools/l2res.py c2 '[dict()]' kv8 | sed 's/^/{"lib": "lazy", "kv8": 1, "r": '$r'} /'
  PDA_LIB_PATH=$A timeout 120 python tools/l2res.py c2 '[dict()]' kv8 | sed 's/^/{"lib": "eager", "kv8": 1, "r": '$r'} /'
done
