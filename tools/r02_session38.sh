#!/bin/bash
# round-2 GPU session 38: why the vertex mode is 3.3x the fused path on the D5a graph — plain tables and
# no L2 hub-row hints, each alone, on the fused path
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s38_build.log 2>&1
B="python bench.py --graph gs22 --template u15-1 --steps 3 --warmup 3 --no-cpu-baseline"
timeout 900 $B --layout anchored_plain > gpurun_out/s38_plain.json 2> gpurun_out/s38_plain.err
SG2V_HINT=0 timeout 900 $B > gpurun_out/s38_nohint.json 2> gpurun_out/s38_nohint.err
SG2V_HINT=0 timeout 900 $B --layout anchored_plain > gpurun_out/s38_plain_nohint.json 2> gpurun_out/s38_plain_nohint.err
python tools/bsum.py gpurun_out/s38_*.json
