# A/B: e4m3 path, working tree (NEW) vs ab_old/libpda.so (OLD), interleaved
for r in 1 2; do
  for spec in "c2 kv8" "c3 kv8" "c5 kv8" "c4_b64_ctx4096 kv8" "c4_b256_ctx32768 kv8" "c4_b16_ctx4096 kv8"; do
    set -- $spec
    echo "NEW $1 $2 $(python tools/psweep.py $1 '[dict()]' $2 | tail -1)"
    echo "OLD $1 $2 $(PDA_LIB_PATH=ab_old/libpda.so python tools/psweep.py $1 '[dict()]' $2 | tail -1)"
  done
done
