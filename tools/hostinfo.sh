mkdir -p gpurun_out
(free -g; echo; nproc; echo; lscpu; echo; cat /proc/meminfo | head -5; nvidia-smi) > gpurun_out/hostinfo.txt 2>&1
python -c "import os; print(os.sched_getaffinity(0))" >> gpurun_out/hostinfo.txt 2>&1
