for r in 1 2; do
for c in u_128_8_1_128_8192_bf16 u_148_8_1_128_8192_bf16 u_74_8_1_128_16384_bf16 u_296_8_1_128_4096_bf16 u_64_4_4_128_4096_fp16 u_74_4_4_128_4096_fp16; do
  timeout 120 python tools/l2res.py $c '[dict(), dict(partition_tokens=4096), dict(partition_tokens=2048)]'
done
done
