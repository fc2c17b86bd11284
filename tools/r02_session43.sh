#!/bin/bash
# round-2 GPU session 43 (final sources with the colour-grouped order): GPU suite, bench contract line,
# ncu DRAM traffic stamped with the final hash, launch list, sweep, smoke
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s43_build.log 2>&1
timeout 900 python bench.py > gpurun_out/s43_bench0.json 2> gpurun_out/s43_bench0.err
python tools/bsum.py gpurun_out/s43_bench0.json
timeout 2700 python -m pytest tests -m gpu -q > gpurun_out/s43_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/s43_tests.log
grep -E "passed|failed|FAILED" gpurun_out/s43_tests.log | tail -6
bash tools/traffic.sh r02final3 u15-1 f32 anchored; echo "traffic rc=$?"
cp gpurun_out/ncu_traffic.json profiles/ncu_traffic.json
timeout 900 python bench.py > gpurun_out/s43_bench.json 2> gpurun_out/s43_bench.err
python tools/bsum.py gpurun_out/s43_bench.json
python -c "import json; d=json.loads(open('gpurun_out/s43_bench.json').read().strip().splitlines()[-1]); r=d['roofline']; print(d['value'], d['e2e']['value'], r['frac'], r['traffic'], r['frac_dram'], d['gpu_launches'], d['clocks'], d['cpu_baseline']['value'])"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s43_launches_bench.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/s43_ncu_bench.log 2>&1; echo "launch list rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s43_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python tools/sweep_templates.py > gpurun_out/s43_sweep.jsonl 2> gpurun_out/s43_sweep.err
cut -c1-120 gpurun_out/s43_sweep.jsonl
