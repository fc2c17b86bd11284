#!/bin/bash
# round-2 GPU session 24: 512-thread CTAs for V-row eMA steps that fill the SM's shared memory (u17 F64)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s24_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_ring.py -x -q > gpurun_out/s24_ring_tests.log 2>&1; echo "ring tests rc=$?" >> gpurun_out/s24_ring_tests.log
tail -3 gpurun_out/s24_ring_tests.log
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 900 $B --template u17 --precision f64 > gpurun_out/s24_u17_f64.json 2> gpurun_out/s24_u17_f64.err
SG2V_EMA512=0 timeout 900 $B --template u17 --precision f64 > gpurun_out/s24_u17_f64_ema256.json 2> gpurun_out/s24_u17_f64_ema256.err
timeout 900 $B --template u17 --precision f32 > gpurun_out/s24_u17_f32.json 2> gpurun_out/s24_u17_f32.err
timeout 900 $B --template u16-2 --precision f64 > gpurun_out/s24_u16-2_f64.json 2> gpurun_out/s24_u16-2_f64.err
SG2V_EMA512=0 timeout 900 $B --template u16-2 --precision f64 > gpurun_out/s24_u16-2_f64_ema256.json 2> gpurun_out/s24_u16-2_f64_ema256.err
python tools/bsum.py gpurun_out/s24_*.json
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/s24_*.json')):
    try: d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, d.get('gpu_launches'), d.get('ema',{}).get('step'), d.get('ema',{}).get('terms_per_s'), d.get('ema',{}).get('frac_smem'))
    except Exception as e: print(f, e)
PY
