# A/B: working tree (NEW) vs build_ab/old (a full older tree with its own libpda.so), interleaved
for r in 1 2; do
  for spec in "c3 kv8" "c2 kv8" "c4_b64_ctx512 fp" "c4_b16_ctx512 fp" "c4_b64_ctx4096 kv8"; do
    set -- $spec
    echo "NEW $1 $2 $(python tools/psweep.py $1 '[dict()]' $2 | tail -1)"
    echo "OLD $1 $2 $(cd build_ab/old && python tools/psweep.py $1 '[dict()]' $2 | tail -1)"
  done
done
