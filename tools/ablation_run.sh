# Prefetch ablation under ncu (paper Table 3 rows), one launch per variant, three configs.
M=$(cat tools/ablation_metrics.txt)
for c in c2 c4_b4_ctx32768 c3; do
  ncu --metrics $M --clock-control none --csv -k regex:'paper_kernel|splitk_kernel' \
      --log-file gpurun_out/ablation_$c.csv python tools/ablation_launches.py --config $c > /dev/null 2>&1
done
ls -la gpurun_out/ablation_*
