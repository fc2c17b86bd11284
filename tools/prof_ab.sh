#!/bin/bash
# per-launch ncu metrics of one colouring for library builds / layouts (A/B experiments)
# tools/prof_ab.sh <tag> <template> <prec>
tag=$1; t=$2; prec=$3
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct
for arm in A Aplain B; do
  lay=anchored; unset SG2V_LIB
  [ $arm = Aplain ] && lay=anchored_plain
  [ $arm = B ] && export SG2V_LIB=ab_old/libsg2v_head.so
  timeout 600 ncu --metrics $M --clock-control none -k regex:astep --csv --log-file gpurun_out/${tag}_${t}_${arm}.csv \
    python tools/prof_one.py $t $prec $lay > gpurun_out/${tag}_${t}_${arm}.log 2>&1
done
