# A/B: tail-only masking (NEW, working tree) vs the previous libpda.so (OLD, ab_old/), interleaved
for r in 1 2; do
  for spec in "c2 kv8" "c3 kv8" "c4_b64_ctx4096 kv8" "c5 kv8" "c2 fp" "c3 fp" "c4_b64_ctx4096 fp" "c4_b256_ctx512 fp"; do
    set -- $spec
    echo "NEW $1 $2 $(python tools/psweep.py $1 '[dict()]' $2 | tail -1)"
    echo "OLD $1 $2 $(PDA_LIB_PATH=ab_old/libpda.so python tools/psweep.py $1 '[dict()]' $2 | tail -1)"
  done
done
