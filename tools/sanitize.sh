# compute-sanitizer over the split-K parity tests small enough for an instrumented run
SEL='(test_parity_vs_oracle and (c1_tiny or gqa16 or zero or gqa4)) or test_kv8_parity_vs_oracle or test_multi_token_parity_vs_oracle or test_fused_append_attention_vs_oracle or test_fused_append_e4m3 or test_cluster_merge_bitwise_equals_combine or test_needle_every_position or test_nan_poison_never_leaks or test_kv8_context_one_is_scaled_v_row'
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -k "$SEL" > gpurun_out/san_$tool.txt 2>&1
  echo "$tool exit=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|passed|failed' gpurun_out/san_$tool.txt | tail -3 | tr '\n' ' ')"
done
