# balanced (persistent, equal blocks per CTA) vs the split-K default on the
# cells below 6.4 TB/s in round 1 and on the BASELINE configs
for cell in u_128_8_1_128_8192_bf16 u_128_32_2_128_8192_bf16 u_32_28_4_128_8192_bf16 c4_b64_ctx4096 \
            u_128_32_32_128_8192_bf16 c4_b16_ctx4096 c4_b4_ctx32768 c4_b256_ctx4096 c2 c3; do
  python tools/psweep.py $cell '[dict(), dict(kernel="balanced"), dict(kernel="balanced", smem_stages=4), dict(kernel="balanced", smem_stages=12)]'
done
