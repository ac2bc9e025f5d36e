# End-of-round measurement set (one B200): bench lines, the bench launch list,
# and one full ncu capture of the C2 split-K kernel.  Outputs in gpurun_out/.
set -x
python bench.py > gpurun_out/end_bench_c2.json 2> gpurun_out/end_bench_c2.err
python bench.py --config c3 --no-extras > gpurun_out/end_bench_c3.json 2>/dev/null
python bench.py --config c5 --no-extras > gpurun_out/end_bench_c5.json 2>/dev/null
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/end_launches_c2.csv \
    python bench.py --steps 2 --warmup 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:splitk_kernel -s 2 -c 1 \
    -o gpurun_out/end_prof_c2 python tools/one_step.py c2 > /dev/null 2>&1
ls -la gpurun_out
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/end_bench_reference.json 2> gpurun_out/end_bench_reference.err
ncu --set full --clock-control none --import-source on -k regex:splitk_kernel -s 2 -c 1 \
    -o gpurun_out/end_prof_c2_kv8 python tools/one_step.py c2 "{}" kv8 > /dev/null 2>&1
python tools/timeline.py c2 > gpurun_out/end_timeline.jsonl 2>/dev/null
python tools/timeline.py c2 "{}" kv8 >> gpurun_out/end_timeline.jsonl 2>/dev/null
python tools/timeline.py c4_b64_ctx4096 >> gpurun_out/end_timeline.jsonl 2>/dev/null
