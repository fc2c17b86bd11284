#!/bin/bash
# round-2 GPU session 33: 8 interleaved rows per 512-thread V-row eMA group (SG2V_EMA512=3) A/B, F32
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s33_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_ring.py -x -q -k vrow > gpurun_out/s33_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/s33_tests.log
tail -2 gpurun_out/s33_tests.log
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --precision f32"
for t in u17 u14-2 u16-2 u13-2; do
  timeout 900 $B --template $t > gpurun_out/s33_${t}.json 2> gpurun_out/s33_${t}.err
  SG2V_EMA512=3 timeout 900 $B --template $t > gpurun_out/s33_${t}_emav8.json 2> gpurun_out/s33_${t}_emav8.err
done
python tools/bsum.py gpurun_out/s33_*.json
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/s33_*.json')):
    try: d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, round(d['value'],4), d.get('ema',{}).get('step'), d.get('ema',{}).get('terms_per_s'), d.get('ema',{}).get('frac_smem'))
    except Exception as e: print(f, e)
PY
