timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r1s21_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r1s21_pytest_gpu.log
ARMS="D" tools/abx.sh r1s21 u16-1 u17-1 u15-1 u12-1
timeout 2400 ncu --replay-mode application --set full --import-source on --clock-control none -k regex:astep -s 6 -c 1 -o gpurun_out/r1s21_top_u15-1 python tools/prof_one.py u15-1 f32 > gpurun_out/r1s21_ncu_full.log 2>&1
