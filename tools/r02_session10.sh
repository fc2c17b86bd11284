#!/bin/bash
# round-2 GPU session 10: launch-configuration A/B for the narrow steps of u15-1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s10_build.log 2>&1
for arm in "D:" "T1:SG2V_TUNE=1" "B128:SG2V_BULK_MIN=128" "HF3:SG2V_HOTFRAC=0.3" "HF12:SG2V_HOTFRAC=1.2" "KB96:SG2V_BULK_KB=96"; do
  tag=${arm%%:*}; kv=${arm#*:}
  env $kv timeout 900 python bench.py --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/s10_$tag.json 2> gpurun_out/s10_$tag.err
  python -c "
import json; d=json.loads(open('gpurun_out/s10_$tag.json').read().strip().splitlines()[-1])
print('$tag', round(d['value'],4), [(s['launch'][:8], round(s['ms'],1)) for s in d['steps_per_colouring'] if s['ms']>1])"
done
