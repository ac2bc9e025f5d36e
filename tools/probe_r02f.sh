for c in c2 u_128_8_1_128_8192_bf16; do
  PDA_LIB_PATH=build_ab/tc_stamps/libpda.so timeout 120 python tools/tc_stamps.py $c
  PDA_LIB_PATH=build_ab/tc_stamps/libpda.so timeout 120 python tools/tc_stamps.py $c l2
done
