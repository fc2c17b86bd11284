#!/bin/bash
# DRAM traffic per launch of one colouring of the bench configuration (ncu, application
# replay so the ~180 GB workspace is not saved per pass) -> profiles/ncu_traffic.json,
# stamped with the library's source hash.   tools/traffic.sh <tag> [template] [precision] [layout]
tag=$1; t=${2:-u15-1}; prec=${3:-f32}; lay=${4:-anchored}
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct
timeout 1200 ncu --metrics $M --replay-mode application --clock-control none \
  -k regex:"colorize|bucket|hist|step|top|reduce" --csv --log-file gpurun_out/traffic_${tag}_${t}_${prec}.csv \
  python tools/prof_one.py $t $prec $lay > gpurun_out/traffic_${tag}_${t}_${prec}.log 2>&1
python tools/traffic_json.py gpurun_out/traffic_${tag}_${t}_${prec}.csv $t $prec $lay 20 --steps gpurun_out/traffic_${tag}_${t}_${prec}.log --out gpurun_out/ncu_traffic.json
