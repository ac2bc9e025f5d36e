# balanced kernel with the warp-uniform refill issue vs split-K (library default), interleaved per cell
for c in u_128_8_1_128_8192_bf16 u_128_32_2_128_8192_bf16 u_32_28_4_128_8192_bf16 c4_b64_ctx4096 c4_b16_ctx8192 c4_b16_ctx16384 c4_b32_ctx8192 c4_b16_ctx4096 c4_b4_ctx32768 u_128_32_32_128_8192_bf16; do
  timeout 300 python tools/psweep.py $c '[dict(), dict(kernel="balanced")]'
done
