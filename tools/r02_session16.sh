#!/bin/bash
# round-2 GPU session 16: warp-per-row register gather (astep_wrow_kernel) + CTA-per-row bucket for hubs
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s16_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_ring.py -x -q > gpurun_out/s16_ring_tests.log 2>&1; echo "ring tests rc=$?" >> gpurun_out/s16_ring_tests.log
tail -3 gpurun_out/s16_ring_tests.log
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
timeout 600 $B > gpurun_out/s16_u15-1.json 2> gpurun_out/s16_u15-1.err
SG2V_WROW=0 timeout 600 $B > gpurun_out/s16_u15-1_wrow0.json 2> gpurun_out/s16_u15-1_wrow0.err
SG2V_WROW_U=2 timeout 600 $B > gpurun_out/s16_u15-1_u2.json 2> gpurun_out/s16_u15-1_u2.err
SG2V_WROW_U=4 timeout 600 $B > gpurun_out/s16_u15-1_u4.json 2> gpurun_out/s16_u15-1_u4.err
SG2V_WROW_U=3 timeout 600 $B > gpurun_out/s16_u15-1_u3.json 2> gpurun_out/s16_u15-1_u3.err
SG2V_WROW_MIN=1 timeout 600 $B > gpurun_out/s16_u15-1_min1.json 2> gpurun_out/s16_u15-1_min1.err
for t in u12-1 u13-1 u14-2; do
  timeout 600 python bench.py --template $t --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s16_$t.json 2> gpurun_out/s16_$t.err
  SG2V_WROW=0 timeout 600 python bench.py --template $t --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s16_${t}_wrow0.json 2> gpurun_out/s16_${t}_wrow0.err
done
python tools/bsum.py gpurun_out/s16_*.json
du -sh gpurun_out
