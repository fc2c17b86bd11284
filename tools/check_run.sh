#!/bin/bash
# GPU parity suite against the check build (device bounds checks; compute-sanitizer is not
# available on the GPU pool): builds lib/libsg2v_check.so and runs the oracle-parity tests with it.
mkdir -p gpurun_out
python -m paper_2009_11665_b200.build --check > gpurun_out/check_build.log 2>&1 || { echo "check build failed"; exit 1; }
SG2V_LIB=$(pwd)/paper_2009_11665_b200/lib/libsg2v_check.so timeout 2400 python -m pytest -q \
  tests/test_gpu_ring.py tests/test_gpu_parity.py tests/test_gpu_variants.py tests/test_gpu_vpart.py \
  > gpurun_out/check_tests.log 2>&1
echo "check-build tests rc=$?" >> gpurun_out/check_tests.log
tail -3 gpurun_out/check_tests.log
