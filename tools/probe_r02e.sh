export L2RES_ONCE=1
ncu --set full --clock-control none --import-source on -k regex:tc_kernel -s 1 -c 1 -o gpurun_out/r02_tc_l2res python tools/l2res.py c2 '[dict(kernel="tc")]' > /dev/null 2>&1
ls -la gpurun_out
