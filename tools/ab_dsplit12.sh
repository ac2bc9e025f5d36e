# split kernel: 8- vs 12-stage ring on one-wave cells (12 stages: 96 KiB in flight per CTA, 2 CTAs/SM)
for c in u_128_8_1_128_8192_bf16 u_64_4_4_128_4096_fp16 c4_b4_ctx32768 u_32_28_4_128_8192_bf16 u_1_32_32_128_32768_bf16 u_128_32_2_128_8192_bf16 c4_b16_ctx4096; do
  timeout 200 python tools/psweep.py $c '[dict(prefetch="off"), dict(prefetch="off", smem_stages=12)]'
done
