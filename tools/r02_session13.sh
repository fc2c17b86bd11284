#!/bin/bash
# round-2 GPU session 13 (after container restore): re-check HEAD — bench u15-1, u12-1/u13-1 narrow steps, GPU tests
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s13_build.log 2>&1
timeout 900 python bench.py > gpurun_out/s13_bench.json 2> gpurun_out/s13_bench.err
for t in u12-1 u13-1 u14-2; do
  timeout 600 python bench.py --template $t --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s13_$t.json 2> gpurun_out/s13_$t.err
done
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/s13_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/s13_tests.log
grep -E "passed|failed|FAILED" gpurun_out/s13_tests.log | tail -8
for f in s13_bench s13_u12-1 s13_u13-1 s13_u14-2; do python -c "
import json; d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1])
print('$f', round(d['value'],4), d.get('status'), [(s['launch'][:22], round(s['ms'],1), round(s.get('frac',0),2)) for s in d['steps_per_colouring'] if s['ms']>0.5])"; done
