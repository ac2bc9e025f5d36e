# compute-sanitizer after the session-3 changes to split-K (start-up: ids / tensor maps / barrier init at
# entry) and the combine kernel (loads up front): parity tests over split-K (plain, tile split, cluster and
# combine merges, e4m3, multi-token) and the planner's small-grid plans
SEL='(parity_vs_oracle or cluster or combine or split_sizes or kv8_parity or multi_token or small or planner) and not full_size and not balanced and not stream and not tc'
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -k "$SEL" > gpurun_out/san_r02d_$tool.txt 2>&1
  echo "$tool exit=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|passed|failed' gpurun_out/san_r02d_$tool.txt | tail -3 | tr '\n' ' ')"
done
