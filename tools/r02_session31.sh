#!/bin/bash
# round-2 GPU session 31: parity suite against the check build (device bounds checks); ncu DRAM traffic
# of the final sources; bench contract line
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s31_build.log 2>&1
bash tools/check_run.sh
bash tools/traffic.sh r02x u15-1 f32 anchored; echo "traffic rc=$?"
timeout 900 python bench.py > gpurun_out/s31_bench.json 2> gpurun_out/s31_bench.err
python tools/bsum.py gpurun_out/s31_bench.json
python -c "import json; d=json.loads(open('gpurun_out/s31_bench.json').read().strip().splitlines()[-1]); print(d['roofline'])"
