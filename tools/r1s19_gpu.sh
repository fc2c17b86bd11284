set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r1s19_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r1s19_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r1s19_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/r1s19_bench.json 2> gpurun_out/r1s19_bench.err
timeout 1200 python tools/sweep_templates.py > gpurun_out/r1s19_sweep.jsonl 2> gpurun_out/r1s19_sweep.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r1s19_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r1s19_ncu_bench.log 2>&1
timeout 900 ncu --replay-mode application --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:astep --csv --log-file gpurun_out/r1s19_traffic_u15-1.csv python tools/prof_one.py u15-1 f32 > gpurun_out/r1s19_prof.log 2>&1
