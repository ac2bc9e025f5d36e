for c in u_128_32_2_128_8192_bf16 u_128_8_1_128_8192_bf16 c4_b64_ctx4096 c4_b16_ctx4096 c2; do
  python tools/l2res.py $c '[dict(), dict(smem_stages=4), dict(smem_stages=12)]'
done
for c in c2 c3 c4_b64_ctx4096; do python tools/l2res.py $c '[dict()]' kv8; done
bash tools/ab_contig.sh
