# compute-sanitizer over the round-2 kernels' GPU tests: the tcgen05 kernel (small shapes, 3 grid sizes,
# forced rescale), the tile-split kernel (g = 16 parity cases) and the prefetch AUTO path (paper kernel)
SEL='test_tc_kernel_vs_oracle or test_tc_kernel_rescale_paths or (test_parity_vs_oracle and gqa16) or test_prefetch_auto_policy_vs_oracle'
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -k "$SEL" > gpurun_out/san_r02_$tool.txt 2>&1
  echo "$tool exit=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|passed|failed' gpurun_out/san_r02_$tool.txt | tail -3 | tr '\n' ' ')"
done
