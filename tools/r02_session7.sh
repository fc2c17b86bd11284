#!/bin/bash
# round-2 GPU session 7: tests (bucket rewrite, bulk fallback), bench u15-1 / u17, template sweep
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s7_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/s7_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/s7_tests.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s7_bench.json 2> gpurun_out/s7_bench.err
timeout 900 python bench.py --template u17 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/s7_u17.json 2> gpurun_out/s7_u17.err
timeout 2400 python tools/sweep_templates.py > gpurun_out/s7_sweep.jsonl 2> gpurun_out/s7_sweep.err
grep -E "passed|failed|FAILED" gpurun_out/s7_tests.log | tail -8
for f in s7_bench s7_u17; do echo $f; cut -c1-200 gpurun_out/$f.json; tail -n 2 gpurun_out/$f.err; done
cut -c1-150 gpurun_out/s7_sweep.jsonl
