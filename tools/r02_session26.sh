#!/bin/bash
# round-2 GPU session 26 (final check of this build): full GPU suite, bench contract line, vertex mode
# world 1, the reference arm, u12-u17 sweep, ncu DRAM traffic + launch list of the bench command
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s26_build.log 2>&1
timeout 900 python bench.py > gpurun_out/s26_bench.json 2> gpurun_out/s26_bench.err
python tools/bsum.py gpurun_out/s26_bench.json
timeout 900 python bench.py --mode vertex --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s26_vertex1.json 2> gpurun_out/s26_vertex1.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/s26_reference.json 2> gpurun_out/s26_reference.err
tail -c 600 gpurun_out/s26_vertex1.json; echo; tail -c 400 gpurun_out/s26_reference.json; echo
timeout 2700 python -m pytest tests -m gpu -q > gpurun_out/s26_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/s26_tests.log
grep -E "passed|failed|FAILED|Error" gpurun_out/s26_tests.log | tail -12
timeout 1500 python tools/sweep_templates.py > gpurun_out/s26_sweep.jsonl 2> gpurun_out/s26_sweep.err
cat gpurun_out/s26_sweep.jsonl | cut -c1-200
bash tools/traffic.sh r02s u15-1 f32 anchored; echo "traffic rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s26_launches_bench.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/s26_ncu_bench.log 2>&1; echo "launch list rc=$?"
du -sh gpurun_out
