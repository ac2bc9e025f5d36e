# Round-2 end measurement set (one B200): bench lines (C2 with every arm, C3, C5, reference), the bench
# launch list, ncu full captures of the C2 step (16-bit and e4m3) summarised on the box, the shape scan.
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/s3_bench_c2.json 2> gpurun_out/s3_bench_c2.err
python bench.py --config c3 --no-extras > gpurun_out/s3_bench_c3.json 2>/dev/null
python bench.py --config c5 --no-extras > gpurun_out/s3_bench_c5.json 2>/dev/null
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/s3_bench_reference.json 2>/dev/null
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s3_launches_c2.csv \
    python bench.py --steps 2 --warmup 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:splitk_kernel -s 2 -c 1 \
    -o /tmp/s3_prof_c2 -f python tools/one_step.py c2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:splitk_kernel -s 2 -c 1 \
    -o /tmp/s3_prof_c2_kv8 -f python tools/one_step.py c2 "{}" kv8 > /dev/null 2>&1
python tools/ncu_summary.py --rep /tmp/s3_prof_c2.ncu-rep --launches gpurun_out/s3_launches_c2.csv \
    --workload c2_llama2_7b --algo-bytes 4296081664 --tag r02s3_c2
python tools/ncu_summary.py --rep /tmp/s3_prof_c2_kv8.ncu-rep --workload c2_llama2_7b_kv8 \
    --algo-bytes 2148040704 --tag r02s3_c2_kv8
cp profiles/r02s3_c2_ncu.md profiles/r02s3_c2_kv8_ncu.md profiles/ncu_summary.json gpurun_out/
ncu -i /tmp/s3_prof_c2.ncu-rep --page source --csv > gpurun_out/s3_c2_source.csv 2>/dev/null
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3_smoke.log 2>&1; echo smoke_rc=$? >> gpurun_out/s3_smoke.log
python tools/shape_scan.py --out gpurun_out/s3_shape_scan.jsonl > /dev/null 2>&1
ls -la gpurun_out
