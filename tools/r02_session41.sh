#!/bin/bash
# round-2 GPU session 41: lanes per eMA output (SG2V_TPO) A/B on the split eMA (u17 F32 / F64, u14-2)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s41_build.log 2>&1
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
for tp in 0 2 4; do
  SG2V_TPO=$tp timeout 900 $B --template u17 > gpurun_out/s41_u17_tpo$tp.json 2> gpurun_out/s41_u17_tpo$tp.err
  SG2V_TPO=$tp timeout 900 $B --template u14-2 > gpurun_out/s41_u14-2_tpo$tp.json 2> gpurun_out/s41_u14-2_tpo$tp.err
done
SG2V_TPO=2 timeout 900 $B --template u17 --precision f64 > gpurun_out/s41_u17f64_tpo2.json 2> gpurun_out/s41_u17f64_tpo2.err
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/s41_*.json')):
    try: d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, round(d['value'],4), d.get('ema',{}).get('step'), d.get('ema',{}).get('terms_per_s'), d.get('ema',{}).get('frac_smem'))
    except Exception as e: print(f, e)
PY
