# tc kernel: PV issued only when V has landed (non-blocking MMA loop) vs the blocking wait (build_ab/tc_base)
A=build_ab/tc_base/libpda.so
for r in 1 2; do
  for c in c2 u_128_8_1_128_8192_bf16 c4_b64_ctx4096; do
    timeout 120 python tools/l2res.py $c '[dict(kernel="tc")]' | sed 's/^/{"lib": "new", "r": '$r'} /'
    PDA_LIB_PATH=$A timeout 120 python tools/l2res.py $c '[dict(kernel="tc")]' | sed 's/^/{"lib": "base", "r": '$r'} /'
  done
done
timeout 300 python tools/tc_check.py > gpurun_out/r02_tc_check_pv.log 2>&1; tail -3 gpurun_out/r02_tc_check_pv.log
