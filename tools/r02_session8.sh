#!/bin/bash
# round-2 GPU session 8: tests with NB-batched bulk stages; bench A/B (SG2V_BULK_STAGE=0)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s8_build.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s8_bench.json 2> gpurun_out/s8_bench.err
SG2V_BULK_STAGE=0 timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s8_bench_nb1.json 2> gpurun_out/s8_bench_nb1.err
SG2V_BULK_MIN=16 timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s8_bench_min16.json 2> gpurun_out/s8_bench_min16.err
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/s8_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/s8_tests.log
grep -E "passed|failed|FAILED" gpurun_out/s8_tests.log | tail -8
for f in s8_bench s8_bench_nb1 s8_bench_min16; do echo $f; cut -c1-150 gpurun_out/$f.json; tail -n 2 gpurun_out/$f.err; done
