#!/bin/bash
# round-2 GPU session 6: tests after the tile-push fix; u17 (split 32 chunks, stage fill) bench
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s6_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_vpart.py -q -x > gpurun_out/s6_vpart.log 2>&1; echo "vpart rc=$?" >> gpurun_out/s6_vpart.log
timeout 900 python bench.py --template u17 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/s6_u17.json 2> gpurun_out/s6_u17.err
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s6_bench.json 2> gpurun_out/s6_bench.err
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/s6_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/s6_tests.log
grep -E "passed|failed|FAILED" gpurun_out/s6_vpart.log gpurun_out/s6_tests.log | tail -12
for f in s6_u17 s6_bench; do echo $f; cut -c1-200 gpurun_out/$f.json; tail -n 2 gpurun_out/$f.err; done
