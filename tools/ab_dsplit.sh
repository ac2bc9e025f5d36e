# D split (8 warps, two per block, one half of d each) on one-wave one-tile grids vs the 4-warp kernel
for c in u_128_8_1_128_8192_bf16 c4_b16_ctx4096 u_64_4_4_128_4096_fp16 c4_b4_ctx32768 c4_b1_ctx32768 u_32_28_4_128_8192_bf16 u_8_32_32_128_8192_bf16 u_1_32_32_128_32768_bf16 c4_b64_ctx4096; do
  timeout 200 python tools/psweep.py $c '[dict(prefetch="off")]' | sed 's/^/{"split": 1} /'
  PDA_TILE_SPLIT=0 timeout 200 python tools/psweep.py $c '[dict(prefetch="off")]' | sed 's/^/{"split": 0} /'
done
