#!/bin/bash
# round-2 GPU session 28: lane-packed warp rows for narrow gathers (<= 16 vectors) — parity + A/B
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s28_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_ring.py -x -q > gpurun_out/s28_ring_tests.log 2>&1; echo "ring tests rc=$?" >> gpurun_out/s28_ring_tests.log
tail -3 gpurun_out/s28_ring_tests.log
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
for cfg in "rmat1m u15-1" "rmat1m u12-1" "rmat1m u14-2" "rmat1m u13-2" "rmat1m u17" "orkut u10-2" "orkut u12-1" "miami u7-2"; do
  set -- $cfg
  timeout 900 $B --graph $1 --template $2 > gpurun_out/s28_$1_$2.json 2> gpurun_out/s28_$1_$2.err
  SG2V_NARROW=0 timeout 900 $B --graph $1 --template $2 > gpurun_out/s28_$1_$2_narrow0.json 2> gpurun_out/s28_$1_$2_narrow0.err
done
python tools/bsum.py gpurun_out/s28_*.json
