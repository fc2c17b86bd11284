#!/bin/bash
# round-2 GPU session 32: 1024-thread V-row eMA CTAs (SG2V_EMA512=2) A/B on F64 eMA-heavy templates
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s32_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_ring.py -x -q -k vrow > gpurun_out/s32_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/s32_tests.log
tail -2 gpurun_out/s32_tests.log
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --precision f64"
for t in u17 u16-2 u15-2; do
  timeout 900 $B --template $t > gpurun_out/s32_${t}_f64.json 2> gpurun_out/s32_${t}_f64.err
  SG2V_EMA512=2 timeout 900 $B --template $t > gpurun_out/s32_${t}_f64_ema1024.json 2> gpurun_out/s32_${t}_f64_ema1024.err
done
python tools/bsum.py gpurun_out/s32_*.json
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/s32_*.json')):
    try: d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, round(d['value'],4), d.get('ema',{}).get('step'), d.get('ema',{}).get('terms_per_s'), d.get('ema',{}).get('frac_smem'))
    except Exception as e: print(f, e)
PY
