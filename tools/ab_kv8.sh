# A/B of the working tree (NEW) against build_ab/libpda_old.so (OLD), interleaved
V='[dict()]'
for r in 1 2; do
for c in c2 c3 c4_b64_ctx4096; do
  for kv in kv8 fp; do
    echo "NEW $kv $(python tools/psweep.py $c "$V" $kv | tail -1)"
    echo "OLD $kv $(PDA_LIB_PATH=build_ab/libpda_old.so python tools/psweep.py $c "$V" $kv | tail -1)"
  done
done; done
