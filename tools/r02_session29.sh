#!/bin/bash
# round-2 GPU session 29 (final build): bench contract line, full GPU suite, sweep, vertex mode world 1,
# ncu DRAM traffic + launch list of the bench command, compute-sanitizer over every kernel path
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s29_build.log 2>&1
timeout 900 python bench.py > gpurun_out/s29_bench.json 2> gpurun_out/s29_bench.err
python tools/bsum.py gpurun_out/s29_bench.json
timeout 2700 python -m pytest tests -m gpu -q > gpurun_out/s29_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/s29_tests.log
grep -E "passed|failed|FAILED|Error" gpurun_out/s29_tests.log | tail -12
bash tools/traffic.sh r02v u15-1 f32 anchored; echo "traffic rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s29_launches_bench.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/s29_ncu_bench.log 2>&1; echo "launch list rc=$?"
timeout 1500 python tools/sweep_templates.py > gpurun_out/s29_sweep.jsonl 2> gpurun_out/s29_sweep.err
timeout 900 python bench.py --mode vertex --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s29_vertex1.json 2> gpurun_out/s29_vertex1.err
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 2400 $CS --tool memcheck --leak-check no --print-limit 50 python tools/sanitize_run.py > gpurun_out/s29_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/s29_memcheck.log
SG2V_RING=1 SG2V_NARROW=1 timeout 2400 $CS --tool memcheck --leak-check no --print-limit 50 python tools/sanitize_run.py > gpurun_out/s29_memcheck_ring.log 2>&1; echo "memcheck(ring, narrow) rc=$?" >> gpurun_out/s29_memcheck_ring.log
timeout 2400 $CS --tool synccheck --print-limit 50 python tools/sanitize_run.py > gpurun_out/s29_synccheck.log 2>&1; echo "synccheck rc=$?" >> gpurun_out/s29_synccheck.log
timeout 3000 $CS --tool racecheck --racecheck-report analysis --print-limit 50 python tools/sanitize_run.py > gpurun_out/s29_racecheck.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/s29_racecheck.log
for f in s29_memcheck s29_memcheck_ring s29_synccheck s29_racecheck; do echo "== $f"; grep -E "ERROR SUMMARY|sanitize_run|rc=|Hazard" gpurun_out/$f.log | sort | uniq -c | head -8; done
du -sh gpurun_out
