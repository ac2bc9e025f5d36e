# DRAM channel balance (min / avg / max over DRAM units) on C2 vs the one-wave cells
M=gpu__time_duration.sum,dram__bytes.min.per_second,dram__bytes.avg.per_second,dram__bytes.max.per_second,dram__cycles_active.min.pct_of_peak_sustained_elapsed,dram__cycles_active.avg.pct_of_peak_sustained_elapsed,dram__cycles_active.max.pct_of_peak_sustained_elapsed,lts__t_requests_srcunit_ltcfabric.sum,lts__t_requests_srcunit_tex.sum,dram__bytes_read.sum
for c in c2 u_128_8_1_128_8192_bf16 u_8_32_32_128_8192_bf16 u_148_8_1_128_8192_bf16 c3; do
  ncu --metrics $M --clock-control none --csv -k regex:splitk_kernel -s 2 -c 1 python tools/one_step.py $c > gpurun_out/q_i_$c.csv 2>/dev/null
done
PSWEEP_CONTIGUOUS=1 ncu --metrics $M --clock-control none --csv -k regex:splitk_kernel -s 2 -c 1 python tools/one_step.py u_128_8_1_128_8192_bf16 > gpurun_out/q_i_contig.csv 2>/dev/null
