#!/bin/bash
# usage: tools/ncu_quick.sh <tag> <kernel-regex> <python args...>   (runs under gpurun)
tag=$1; shift; kre=$1; shift
M=gpu__time_duration.sum,launch__occupancy_limit_shared_mem,launch__occupancy_limit_registers,launch__grid_size,sm__ctas_launched.sum,sm__warps_active.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_elapsed,launch__shared_mem_per_block_dynamic,launch__registers_per_thread,sm__cycles_elapsed.max,dram__bytes_read.sum,lts__t_sector_op_read_hit_rate.pct
mkdir -p gpurun_out
ncu --metrics $M --clock-control none --csv -k regex:"$kre" -s 1 -c 1 "$@" > gpurun_out/q_$tag.csv 2>/dev/null
