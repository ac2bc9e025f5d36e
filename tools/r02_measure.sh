# Round-2 measurement set (one B200): bench lines (C2 with every arm, C3, C5, reference), the bench
# launch list, ncu full captures of the C2 step (16-bit split-K, e4m3, tc).  Outputs in gpurun_out/.
python bench.py > gpurun_out/r02f_bench_c2.json 2> gpurun_out/r02f_bench_c2.err
python bench.py --config c3 --no-extras > gpurun_out/r02f_bench_c3.json 2>/dev/null
python bench.py --config c5 --no-extras > gpurun_out/r02f_bench_c5.json 2>/dev/null
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02f_bench_reference.json 2>/dev/null
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02f_launches_c2.csv \
    python bench.py --steps 2 --warmup 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:splitk_kernel -s 2 -c 1 \
    -o gpurun_out/r02f_prof_c2 python tools/one_step.py c2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:splitk_kernel -s 2 -c 1 \
    -o gpurun_out/r02f_prof_c2_kv8 python tools/one_step.py c2 "{}" kv8 > /dev/null 2>&1
ls -la gpurun_out | tail -12
