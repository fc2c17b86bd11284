#!/bin/bash
# one launch of a template's step sequence under ncu (application replay: no 100+ GB save/restore)
# tools/ncu_top.sh <tag> <template> <launch index among astep launches> [lib]
tag=$1; t=$2; idx=$3; lib=$4
M=gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct,smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio,launch__registers_per_thread,launch__occupancy_limit_registers,launch__occupancy_limit_shared_mem,launch__grid_size
if [ -n "$lib" ]; then export SG2V_LIB=$lib; fi
timeout 900 ncu --replay-mode application --metrics $M --clock-control none -k regex:astep -s $idx -c 1 --csv \
  --log-file gpurun_out/${tag}_${t}_${idx}.csv python tools/prof_one.py $t f32 > gpurun_out/${tag}_${t}_${idx}.log 2>&1
