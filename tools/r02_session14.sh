#!/bin/bash
# round-2 GPU session 14: where do the narrow gather steps (u15-1 s3-s5) spend their time?
#  (1) per-launch list of one full-size colouring: time, DRAM bytes, instructions, issue / warp occupancy
#  (2) ncu --set full (source) of the s3 / s4 register-gather and s5 bulk launches at RMAT scale 18
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s14_build.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,smsp__inst_executed.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__block_size,launch__registers_per_thread,smsp__issue_active.avg.pct_of_peak_sustained_active
timeout 1500 ncu --metrics $M --replay-mode application --clock-control none \
  -k regex:"colorize|bucket|hist|step|top|reduce" --csv --log-file gpurun_out/s14_launches_u15-1.csv \
  python tools/prof_one.py u15-1 f32 anchored 1 20 > gpurun_out/s14_launches.log 2>&1
echo "launch list rc=$?"
timeout 900 ncu --metrics $M --replay-mode application --clock-control none \
  -k regex:"astep" --csv --log-file gpurun_out/s14_launches_u15-1_s18.csv \
  python tools/prof_one.py u15-1 f32 anchored 1 18 > gpurun_out/s14_launches18.log 2>&1
for idx in 1 3 4; do
  timeout 1500 ncu --set full --import-source on --replay-mode application --clock-control none \
    -k regex:astep -s $idx -c 1 -f -o gpurun_out/s14_full_u15-1_$idx \
    python tools/prof_one.py u15-1 f32 anchored 1 18 > gpurun_out/s14_full_$idx.log 2>&1
  echo "ncu full $idx rc=$?"
done
