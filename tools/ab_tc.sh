timeout 300 python tools/tc_check.py parity
for c in c2 u_128_8_1_128_8192_bf16 c4_b64_ctx4096 c3 u_128_32_2_128_8192_bf16; do
  timeout 120 python tools/l2res.py $c '[dict(kernel="tc"), dict()]'
done
