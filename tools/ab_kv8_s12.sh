# e4m3: 12-stage ring consumed block by block at 4 CTAs/SM vs 16 stages in pairs at 3 CTAs/SM
for c in c2 c3 c5 c4_b64_ctx4096 c4_b256_ctx4096 c4_b16_ctx32768 c4_b1_ctx512 c4_b4_ctx4096 c4_b64_ctx512; do
python tools/psweep.py $c '[dict(), dict(smem_stages=12), dict(smem_stages=8), dict(smem_stages=24)]' kv8
done
