#!/bin/bash
# round-2 GPU session 42: colour-grouped row order for projected-source steps (SG2V_CORDER=1) — parity + A/B
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s42_build.log 2>&1
SG2V_CORDER=1 timeout 1200 python -m pytest tests/test_gpu_ring.py tests/test_gpu_parity.py -x -q > gpurun_out/s42_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/s42_tests.log
tail -2 gpurun_out/s42_tests.log
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
for t in u15-1 u14-1 u13-1; do
  timeout 900 $B --template $t > gpurun_out/s42_$t.json 2> gpurun_out/s42_$t.err
  SG2V_CORDER=1 timeout 900 $B --template $t > gpurun_out/s42_${t}_corder.json 2> gpurun_out/s42_${t}_corder.err
done
SG2V_CORDER=1 timeout 900 $B --template u17 --precision f64 > gpurun_out/s42_u17f64_corder.json 2> gpurun_out/s42_u17f64_corder.err
python tools/bsum.py gpurun_out/s42_*.json
