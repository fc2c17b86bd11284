#!/bin/bash
# round-2 GPU session 17: full GPU suite + bench after the warp-row gather / bucket rewrite
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s17_build.log 2>&1
timeout 900 python bench.py > gpurun_out/s17_bench.json 2> gpurun_out/s17_bench.err
for t in u12-1 u13-1 u14-1 u16-1; do
  timeout 600 python bench.py --template $t --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s17_$t.json 2> gpurun_out/s17_$t.err
done
python tools/bsum.py gpurun_out/s17_*.json
timeout 2700 python -m pytest tests -m gpu -q > gpurun_out/s17_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/s17_tests.log
grep -E "passed|failed|FAILED|Error" gpurun_out/s17_tests.log | tail -12
