#!/bin/bash
# round-2 GPU session 18: ncu DRAM traffic of the bench configuration at HEAD; u17 / u17-1 per-step tables
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s18_build.log 2>&1
bash tools/traffic.sh r02n u15-1 f32 anchored; echo "traffic rc=$?"
for p in f32 f64; do
  timeout 900 python bench.py --template u17 --precision $p --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/s18_u17_$p.json 2> gpurun_out/s18_u17_$p.err
done
timeout 900 python bench.py --template u17-1 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/s18_u17-1.json 2> gpurun_out/s18_u17-1.err
python tools/bsum.py gpurun_out/s18_*.json
