# Prefetch ablation under ncu on the 12-cell batch x context grid (B in {1,16,64,256},
# ctx in {512,4096,32768}; ragged lengths): paper-structure and split-K kernels,
# prefetch off / on (paper Table 3 rows: L2 hit rate, DRAM bytes, long-scoreboard share)
M=$(cat tools/ablation_metrics.txt)
for b in 1 16 64 256; do for c in 512 4096 32768; do
  cfg=c4_b${b}_ctx${c}
  ncu --metrics $M --clock-control none --csv -k regex:'paper_kernel|splitk_kernel' \
      --log-file gpurun_out/ablation_$cfg.csv python tools/ablation_launches.py --grid --config $cfg > /dev/null 2>&1
done; done
ls -la gpurun_out/ablation_*
