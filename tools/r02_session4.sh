#!/bin/bash
# round-2 GPU session 4: tests; bench u15-1 + u17; template sweep; ncu --set full of bulk launches (scale 18)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s4_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/s4_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/s4_tests.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/s4_bench.json 2> gpurun_out/s4_bench.err
timeout 900 python bench.py --template u17 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/s4_u17.json 2> gpurun_out/s4_u17.err
timeout 1800 python tools/sweep_templates.py > gpurun_out/s4_sweep.jsonl 2> gpurun_out/s4_sweep.err
for idx in 3 0; do
  timeout 1200 ncu --set full --import-source on --replay-mode application --clock-control none \
    -k regex:astep_bulk -s $idx -c 1 -f -o gpurun_out/s4_ncu_bulk_$idx \
    python tools/prof_one.py u15-1 f32 anchored 1 18 > gpurun_out/s4_ncu_bulk_$idx.log 2>&1
  echo "ncu $idx rc=$?"
done
tail -n 3 gpurun_out/s4_tests.log
for f in s4_bench s4_u17; do echo $f; cut -c1-300 gpurun_out/$f.json; tail -n 2 gpurun_out/$f.err; done
cat gpurun_out/s4_sweep.jsonl | cut -c1-200
