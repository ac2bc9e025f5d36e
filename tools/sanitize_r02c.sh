# balanced kernel after moving its slot protocol to mbarriers: parity tests, then racecheck + synccheck
timeout 900 python -m pytest tests -m gpu -q -k "balanced" 2>&1 | tail -2
SEL='balanced and not full_size'
for tool in racecheck synccheck memcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -k "$SEL" > gpurun_out/san_r02c_$tool.txt 2>&1
  echo "$tool exit=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|passed|failed' gpurun_out/san_r02c_$tool.txt | tail -3 | tr '\n' ' ')"
done
for c in u_128_8_1_128_8192_bf16 c4_b64_ctx4096 c2; do
  timeout 120 python tools/l2res.py $c '[dict(kernel="balanced")]'
  PDA_LIB_PATH=build_ab/tc_base/libpda.so timeout 120 python tools/l2res.py $c '[dict(kernel="balanced")]' | sed 's/^/{"lib": "atomic-fence"} /'
done
