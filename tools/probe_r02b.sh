# ncu --set full with source (stall sampling) on L2-resident launches: where the consumer chain spends time
export L2RES_ONCE=1
ncu --set full --clock-control none --import-source on -k regex:splitk -s 1 -c 1 -o gpurun_out/r02_l2res_u128_8_1 python tools/l2res.py u_128_8_1_128_8192_bf16 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:splitk -s 1 -c 1 -o gpurun_out/r02_l2res_c2kv8 python tools/l2res.py c2 '[dict()]' kv8 > /dev/null 2>&1
[ -n "$THIRD" ] && ncu --set full --clock-control none --import-source on -k regex:splitk -s 1 -c 1 -o gpurun_out/r02_l2res_u128_32_2 python tools/l2res.py u_128_32_2_128_8192_bf16 > /dev/null 2>&1
ls -la gpurun_out
