# e4m3 two-tile kernel: 3 CTAs/SM (NEW; S16 spills 24 B, S12 none) vs 2 CTAs/SM (OLD, ab_old/)
for r in 1 2; do
  for spec in "c5 2" "c3 4" "u_64_32_2_128_8192_bf16 1" "u_256_32_2_128_8192_bf16 1"; do
    set -- $spec
    echo "NEW $1 q$2 $(python tools/psweep.py $1 '[dict(), dict(smem_stages=12)]' kv8 $2 | tr '\n' ' ' | sed 's/"k_scale[^}]*"us"/"us"/g')"
    echo "OLD $1 q$2 $(PDA_LIB_PATH=ab_old/libpda.so python tools/psweep.py $1 '[dict(), dict(smem_stages=12)]' kv8 $2 | tr '\n' ' ' | sed 's/"k_scale[^}]*"us"/"us"/g')"
  done
done
