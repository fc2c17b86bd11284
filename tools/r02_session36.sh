#!/bin/bash
# round-2 GPU session 36: warp-row gather at 64 registers (8 CTAs) for rows of 17-32 vectors (u15-1 step 4) A/B
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s36_build.log 2>&1
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
timeout 900 $B > gpurun_out/s36_u15-1.json 2> gpurun_out/s36_u15-1.err
SG2V_WROW_MIN=17 timeout 900 $B > gpurun_out/s36_u15-1_min17.json 2> gpurun_out/s36_u15-1_min17.err
SG2V_WROW_MIN=17 SG2V_WROW_U=4 timeout 900 $B > gpurun_out/s36_u15-1_min17u4.json 2> gpurun_out/s36_u15-1_min17u4.err
for t in u14-1 u12-1 u13-1; do
  timeout 900 $B --template $t > gpurun_out/s36_$t.json 2> gpurun_out/s36_$t.err
  SG2V_WROW_MIN=17 SG2V_WROW_U=4 timeout 900 $B --template $t > gpurun_out/s36_${t}_min17u4.json 2> gpurun_out/s36_${t}_min17u4.err
done
python tools/bsum.py gpurun_out/s36_*.json
