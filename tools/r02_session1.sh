#!/bin/bash
# round-2 GPU session 1: smoke, GPU tests, bench A/B (bulk-staged gather on/off), traffic
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s1_build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s1_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/s1_smoke.log
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/s1_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/s1_tests.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s1_bench_bulk.json 2> gpurun_out/s1_bench_bulk.err
SG2V_BULK=0 timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s1_bench_nobulk.json 2> gpurun_out/s1_bench_nobulk.err
bash tools/traffic.sh s1 u15-1 f32 anchored > gpurun_out/s1_traffic.log 2>&1
tail -3 gpurun_out/s1_smoke.log gpurun_out/s1_tests.log; cut -c1-600 gpurun_out/s1_bench_bulk.json gpurun_out/s1_bench_nobulk.json; tail -3 gpurun_out/s1_traffic.log
