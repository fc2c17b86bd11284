#!/bin/bash
# round-2 GPU session 24b: (rerun after the binding fix) 512-thread V-row eMA CTAs, u17 / u16-2; then the GTDIV A/B
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s24_build.log 2>&1
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 900 $B --template u17 --precision f64 > gpurun_out/s24_u17_f64.json 2> gpurun_out/s24_u17_f64.err
SG2V_EMA512=0 timeout 900 $B --template u17 --precision f64 > gpurun_out/s24_u17_f64_ema256.json 2> gpurun_out/s24_u17_f64_ema256.err
timeout 900 $B --template u16-2 --precision f64 > gpurun_out/s24_u16-2_f64.json 2> gpurun_out/s24_u16-2_f64.err
SG2V_EMA512=0 timeout 900 $B --template u16-2 --precision f64 > gpurun_out/s24_u16-2_f64_ema256.json 2> gpurun_out/s24_u16-2_f64_ema256.err
python tools/bsum.py gpurun_out/s24_*.json
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/s24_*.json')):
    try: d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, d.get('gpu_launches'), d.get('ema',{}).get('step'), d.get('ema',{}).get('terms_per_s'), d.get('ema',{}).get('frac_smem'))
    except Exception as e: print(f, e)
PY
bash tools/r02_session25.sh
