#!/bin/bash
# round-2 GPU session 37: Graph500-like scale-22 graph (D5a, n = 4.19M, nnz = 128M): u12-1 / u15-1 fused
# and vertex mode at world 1 (u17 / u20 there need > 1 GPU: DESIGN §8)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s37_build.log 2>&1
B="python bench.py --graph gs22 --steps 3 --warmup 3 --no-cpu-baseline"
timeout 900 $B --template u12-1 > gpurun_out/s37_gs22_u12-1.json 2> gpurun_out/s37_gs22_u12-1.err
timeout 900 $B --template u15-1 > gpurun_out/s37_gs22_u15-1.json 2> gpurun_out/s37_gs22_u15-1.err
timeout 900 $B --template u15-1 --mode vertex > gpurun_out/s37_gs22_u15-1_vertex1.json 2> gpurun_out/s37_gs22_u15-1_vertex1.err
python tools/bsum.py gpurun_out/s37_*.json
tail -c 300 gpurun_out/s37_gs22_u15-1_vertex1.json; tail -3 gpurun_out/s37_gs22_u15-1_vertex1.err
