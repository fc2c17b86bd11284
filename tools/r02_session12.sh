#!/bin/bash
# round-2 GPU session 12: split pipeline for narrower gathers (u14-2, u16-2) A/B; GPU tests
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s12_build.log 2>&1
for t in u14-2 u16-2; do
  timeout 900 python bench.py --template $t --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/s12_$t.json 2> gpurun_out/s12_$t.err
  SG2V_SPLIT=0 timeout 900 python bench.py --template $t --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/s12_${t}_nosplit.json 2> gpurun_out/s12_${t}_nosplit.err
done
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/s12_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/s12_tests.log
grep -E "passed|failed|FAILED" gpurun_out/s12_tests.log | tail -8
for f in s12_u14-2 s12_u14-2_nosplit s12_u16-2 s12_u16-2_nosplit; do python -c "
import json; d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1])
print('$f', round(d['value'],4), d['status'], [(s['launch'][:22], round(s['ms'],1)) for s in d['steps_per_colouring'] if s['ms']>1])"; done
