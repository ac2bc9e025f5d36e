python -m pytest tests -m gpu -x -q > gpurun_out/r02_gputest_c.log 2>&1; echo rc=$? >> gpurun_out/r02_gputest_c.log
bash tools/ab_tile_split.sh > gpurun_out/r02_ab_ts2.log 2>&1
python tools/prefetch_policy_ab.py 50 c1 c4_b1_ctx512 c4_b1_ctx1024 c4_b1_ctx2048 c4_b1_ctx4096 c4_b2_ctx1024 c4_b4_ctx512 c4_b4_ctx2048 c4_b16_ctx512 c4_b1_ctx32768 c4_b4_ctx32768 c4_b16_ctx4096 > gpurun_out/r02_prefetch_policy.jsonl 2> gpurun_out/r02_prefetch_policy.err
python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench_c.json 2> gpurun_out/r02_bench_c.err
