# full ncu of the one-wave 8/1 cell with 8 and 12 ring stages (why the deeper ring is slower)
for v in s8 s12; do
  if [ $v = s8 ]; then O='{}'; else O='{"smem_stages": 12}'; fi
  ncu --set full --clock-control none -k regex:splitk_kernel -s 2 -c 1 -o /tmp/r02h_$v -f python tools/one_step.py u_128_8_1_128_8192_bf16 "$O" > /dev/null 2>&1
  ncu -i /tmp/r02h_$v.ncu-rep --page raw --csv > gpurun_out/r02h_${v}_raw.csv 2>&1
  ncu -i /tmp/r02h_$v.ncu-rep --page details --csv > gpurun_out/r02h_${v}_details.csv 2>&1
done
ls -la gpurun_out/
