#!/bin/bash
# round-2 GPU session 30 (final build, after the row-group smem guard): variants first, then the full
# GPU suite, bench contract line, ncu DRAM traffic + launch list, sweep, vertex mode world 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s30_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_variants.py -x -q > gpurun_out/s30_variants.log 2>&1; echo "variants rc=$?" >> gpurun_out/s30_variants.log
tail -3 gpurun_out/s30_variants.log
timeout 900 python bench.py > gpurun_out/s30_bench.json 2> gpurun_out/s30_bench.err
python tools/bsum.py gpurun_out/s30_bench.json
timeout 2700 python -m pytest tests -m gpu -q > gpurun_out/s30_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/s30_tests.log
grep -E "passed|failed|FAILED|Error" gpurun_out/s30_tests.log | tail -12
bash tools/traffic.sh r02w u15-1 f32 anchored; echo "traffic rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s30_launches_bench.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/s30_ncu_bench.log 2>&1; echo "launch list rc=$?"
timeout 1500 python tools/sweep_templates.py > gpurun_out/s30_sweep.jsonl 2> gpurun_out/s30_sweep.err
timeout 900 python bench.py --mode vertex --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s30_vertex1.json 2> gpurun_out/s30_vertex1.err
du -sh gpurun_out
