# compute-sanitizer after the tc PV change and over the rescale-pattern tests
SEL='test_tc_kernel_vs_oracle or test_tc_kernel_rescale_paths or (test_softmax_rescale_patterns and (steep or needle) and (default or balanced or stream))'
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -k "$SEL" > gpurun_out/san_r02b_$tool.txt 2>&1
  echo "$tool exit=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|passed|failed' gpurun_out/san_r02b_$tool.txt | tail -3 | tr '\n' ' ')"
done
