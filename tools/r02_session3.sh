#!/bin/bash
# round-2 GPU session 3: tests; bench A/B (bulk NC variants for mid rows); u17 eMA (bank schedule on/off)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s3_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/s3_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/s3_tests.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s3_bench.json 2> gpurun_out/s3_bench.err
SG2V_BULK_MIN=128 timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s3_bench_min128.json 2> gpurun_out/s3_bench_min128.err
timeout 900 python bench.py --template u17 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/s3_u17.json 2> gpurun_out/s3_u17.err
SG2V_EMA_SCHED=0 timeout 900 python bench.py --template u17 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/s3_u17_nosched.json 2> gpurun_out/s3_u17_nosched.err
M=gpu__time_duration.sum,smsp__inst_executed.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,launch__registers_per_thread,launch__grid_size
for sch in 1 0; do
  SG2V_EMA_SCHED=$sch timeout 900 ncu --replay-mode application --metrics $M --clock-control none -k regex:astep -s 5 -c 1 --csv \
    --log-file gpurun_out/s3_ncu_u17_ema_sched$sch.csv python tools/prof_one.py u17 f32 anchored 1 > gpurun_out/s3_ncu_u17_$sch.log 2>&1
done
tail -n 3 gpurun_out/s3_tests.log
for f in s3_bench s3_bench_min128 s3_u17 s3_u17_nosched; do echo $f; cut -c1-300 gpurun_out/$f.json; tail -n 2 gpurun_out/$f.err; done
