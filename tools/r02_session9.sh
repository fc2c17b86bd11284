#!/bin/bash
# round-2 GPU session 9: tests (incl. bench contract at N=1 and N=2 torchrun), bench after the revert, u17 M_a staging A/B
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s9_build.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s9_bench.json 2> gpurun_out/s9_bench.err
timeout 900 python bench.py --template u17 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/s9_u17.json 2> gpurun_out/s9_u17.err
SG2V_STAGE_KB=40 timeout 900 python bench.py --template u17 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/s9_u17_stage40.json 2> gpurun_out/s9_u17_stage40.err
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/s9_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/s9_tests.log
grep -E "passed|failed|FAILED" gpurun_out/s9_tests.log | tail -8
for f in s9_bench s9_u17 s9_u17_stage40; do echo $f; cut -c1-150 gpurun_out/$f.json; tail -n 2 gpurun_out/$f.err; done
