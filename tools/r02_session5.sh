#!/bin/bash
# round-2 GPU session 5: tests (all, no -x), bench u15-1 (+cpu baseline), u17 split A/B, sweep,
# ncu --set full of the bulk top / step-5 launches summarised in place (the .ncu-rep files are
# deleted: gpurun_out must stay under 64 MiB)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s5_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/s5_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/s5_tests.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/s5_bench.json 2> gpurun_out/s5_bench.err
timeout 900 python bench.py --template u17 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/s5_u17.json 2> gpurun_out/s5_u17.err
SG2V_SPLIT=0 timeout 900 python bench.py --template u17 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/s5_u17_nosplit.json 2> gpurun_out/s5_u17_nosplit.err
timeout 900 python bench.py --template u14-2 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/s5_u14-2.json 2> gpurun_out/s5_u14-2.err
SG2V_SPLIT=0 timeout 900 python bench.py --template u14-2 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/s5_u14-2_nosplit.json 2> gpurun_out/s5_u14-2_nosplit.err
for idx in 3 0; do
  timeout 1200 ncu --set full --import-source on --replay-mode application --clock-control none \
    -k regex:astep_bulk -s $idx -c 1 -f -o /tmp/s5_ncu_bulk_$idx \
    python tools/prof_one.py u15-1 f32 anchored 1 18 > gpurun_out/s5_ncu_bulk_$idx.log 2>&1
  echo "ncu $idx rc=$?"
  python tools/ncu_summary.py /tmp/s5_ncu_bulk_$idx.ncu-rep > gpurun_out/s5_ncu_bulk_$idx.json 2>&1
  ncu -i /tmp/s5_ncu_bulk_$idx.ncu-rep --page source --csv > /tmp/s5_src_$idx.csv 2>/dev/null; head -c 3000000 /tmp/s5_src_$idx.csv > gpurun_out/s5_ncu_bulk_${idx}_source.csv
  rm -f /tmp/s5_ncu_bulk_$idx.ncu-rep
done
du -sh gpurun_out
grep -E "passed|failed|FAILED|Error" gpurun_out/s5_tests.log | tail -15
for f in s5_bench s5_u17 s5_u17_nosplit s5_u14-2 s5_u14-2_nosplit; do echo $f; cut -c1-200 gpurun_out/$f.json; tail -n 2 gpurun_out/$f.err; done
