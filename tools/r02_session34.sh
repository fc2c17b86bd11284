#!/bin/bash
# round-2 GPU session 34 (final sources): ncu DRAM traffic stamped with the final source hash, bench
# contract line, full GPU suite, launch list of the bench command
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s34_build.log 2>&1
bash tools/traffic.sh r02final u15-1 f32 anchored; echo "traffic rc=$?"
cp gpurun_out/ncu_traffic.json profiles/ncu_traffic.json
timeout 900 python bench.py > gpurun_out/s34_bench.json 2> gpurun_out/s34_bench.err
python tools/bsum.py gpurun_out/s34_bench.json
python -c "import json; d=json.loads(open('gpurun_out/s34_bench.json').read().strip().splitlines()[-1]); r=d['roofline']; print(r['frac'], r['traffic'], r['frac_dram'], r['traffic_source'], d['gpu_launches'], d['clocks'])"
timeout 2700 python -m pytest tests -m gpu -q > gpurun_out/s34_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/s34_tests.log
grep -E "passed|failed|FAILED" gpurun_out/s34_tests.log | tail -6
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s34_launches_bench.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/s34_ncu_bench.log 2>&1; echo "launch list rc=$?"
