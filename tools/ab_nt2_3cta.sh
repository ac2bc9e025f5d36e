# A/B: two-tile 16-bit split-K at 3 CTAs/SM (NEW, 166 registers) vs 2 (OLD, ab_old/)
for r in 1 2; do
  for spec in "c3 4" "c3 3" "c5 2" "c2 16" "u_512_32_2_128_1024_bf16 1" "u_128_32_2_128_32768_bf16 1" "u_512_32_2_128_8192_bf16 1" "u_64_32_2_128_8192_bf16 1"; do
    set -- $spec
    echo "NEW $1 q$2 $(python tools/psweep.py $1 '[dict()]' fp $2 | tail -1)"
    echo "OLD $1 q$2 $(PDA_LIB_PATH=ab_old/libpda.so python tools/psweep.py $1 '[dict()]' fp $2 | tail -1)"
  done
done
