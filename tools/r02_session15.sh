#!/bin/bash
# round-2 GPU session 15: self-fed warp-ring gather (astep_ring_kernel) — parity, A/B, gather roofline
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s15_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_ring.py -x -q > gpurun_out/s15_ring_tests.log 2>&1; echo "ring tests rc=$?" >> gpurun_out/s15_ring_tests.log
tail -3 gpurun_out/s15_ring_tests.log
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
timeout 600 $B > gpurun_out/s15_u15-1.json 2> gpurun_out/s15_u15-1.err
SG2V_RING=0 timeout 600 $B > gpurun_out/s15_u15-1_ring0.json 2> gpurun_out/s15_u15-1_ring0.err
SG2V_RING_MAX=256 timeout 600 $B > gpurun_out/s15_u15-1_ringmax256.json 2> gpurun_out/s15_u15-1_ringmax256.err
SG2V_RING_KB=32 timeout 600 $B > gpurun_out/s15_u15-1_ringkb32.json 2> gpurun_out/s15_u15-1_ringkb32.err
SG2V_RING_KB=8 timeout 600 $B > gpurun_out/s15_u15-1_ringkb8.json 2> gpurun_out/s15_u15-1_ringkb8.err
for t in u12-1 u13-1; do
  timeout 600 python bench.py --template $t --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s15_$t.json 2> gpurun_out/s15_$t.err
done
python tools/bsum.py gpurun_out/s15_*.json
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o gpurun_out/gather_roof tools/gather_roof.cu && timeout 600 gpurun_out/gather_roof 24 > gpurun_out/s15_gather_roof.json 2>&1
cat gpurun_out/s15_gather_roof.json
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,smsp__inst_executed.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__block_size,launch__registers_per_thread,smsp__issue_active.avg.pct_of_peak_sustained_active
timeout 1500 ncu --metrics $M --replay-mode application --clock-control none \
  -k regex:"colorize|bucket|hist|step|top|reduce" --csv --log-file gpurun_out/s15_launches_u15-1.csv \
  python tools/prof_one.py u15-1 f32 anchored 1 20 > gpurun_out/s15_launches.log 2>&1
echo "launch list rc=$?"
rm -f gpurun_out/gather_roof
du -sh gpurun_out
