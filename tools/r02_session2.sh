#!/bin/bash
# round-2 GPU session 2: GPU tests, bench (bulk wide + heavy narrow), traffic, ncu full of narrow steps
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s2_build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/s2_smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/s2_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/s2_tests.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s2_bench.json 2> gpurun_out/s2_bench.err
SG2V_HEAVY=0 timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s2_bench_noheavy.json 2> gpurun_out/s2_bench_noheavy.err
timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --mode vertex > gpurun_out/s2_bench_vertex.json 2> gpurun_out/s2_bench_vertex.err
bash tools/traffic.sh s2 u15-1 f32 anchored > gpurun_out/s2_traffic.log 2>&1
tail -n 3 gpurun_out/s2_smoke.log gpurun_out/s2_tests.log
for f in s2_bench s2_bench_noheavy s2_bench_vertex; do echo $f; cut -c1-400 gpurun_out/$f.json; tail -n 3 gpurun_out/$f.err; done
tail -n 3 gpurun_out/s2_traffic.log
