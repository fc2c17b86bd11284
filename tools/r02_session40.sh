#!/bin/bash
# round-2 GPU session 40 (final sources after the world-1 whole-row fix): vertex mode on the D5a graph,
# GPU suite, ncu DRAM traffic stamped with the final hash, bench contract line, launch list
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s40_build.log 2>&1
timeout 900 python bench.py --graph gs22 --template u15-1 --mode vertex --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s40_gs22_vertex1.json 2> gpurun_out/s40_gs22_vertex1.err
timeout 900 python bench.py --mode vertex --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s40_vertex1.json 2> gpurun_out/s40_vertex1.err
python -c "
import json
for f in ['gpurun_out/s40_gs22_vertex1.json','gpurun_out/s40_vertex1.json']:
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, d['value'], d['kernel_ms_per_step'])"
bash tools/traffic.sh r02final2 u15-1 f32 anchored; echo "traffic rc=$?"
cp gpurun_out/ncu_traffic.json profiles/ncu_traffic.json
timeout 900 python bench.py > gpurun_out/s40_bench.json 2> gpurun_out/s40_bench.err
python tools/bsum.py gpurun_out/s40_bench.json
python -c "import json; d=json.loads(open('gpurun_out/s40_bench.json').read().strip().splitlines()[-1]); r=d['roofline']; print(d['value'], d['e2e']['value'], r['frac'], r['traffic'], r['frac_dram'], d['gpu_launches'], d['clocks'])"
timeout 2700 python -m pytest tests -m gpu -q > gpurun_out/s40_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/s40_tests.log
grep -E "passed|failed|FAILED" gpurun_out/s40_tests.log | tail -6
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s40_launches_bench.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/s40_ncu_bench.log 2>&1; echo "launch list rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s40_smoke.log 2>&1; echo "smoke rc=$?"
