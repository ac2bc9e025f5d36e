# tile-split kernel (8 consumer warps, one head tile each; default for two-tile
# 16-bit steps) vs the two-tile 4-warp kernel (PDA_TILE_SPLIT=0), ring depths
for c in u_128_32_2_128_8192_bf16 u_32_32_2_128_8192_bf16 u_256_32_2_128_4096_bf16 u_16_32_2_128_32768_bf16 u_64_64_4_128_8192_bf16; do
  python tools/psweep.py $c '[dict(), dict(smem_stages=8)]' | sed 's/^/{"ts": 1} /'
  PDA_TILE_SPLIT=0 python tools/psweep.py $c '[dict()]' | sed 's/^/{"ts": 0} /'
done
for cq in "c3 4" "c2 16" "c5 2"; do set -- $cq
  python tools/psweep.py $1 '[dict(), dict(smem_stages=8)]' "" $2 | sed 's/^/{"ts": 1} /'
  PDA_TILE_SPLIT=0 python tools/psweep.py $1 '[dict()]' "" $2 | sed 's/^/{"ts": 0} /'
done
