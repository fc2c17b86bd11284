timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r1s32_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r1s32_pytest_gpu.log
python tools/vcheck.py default u15-2,u16-2 f32 > gpurun_out/r1s32_vcheck.txt 2>&1; SG2V_TUNE=9 python tools/vcheck.py forceV4 u15-2,u16-2,u15-1 f32 >> gpurun_out/r1s32_vcheck.txt 2>&1
ARMS="D B" LIBB=ab_old/libsg2v_c2.so tools/abx.sh r1s32 u15-1 u17
