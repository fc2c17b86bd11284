#!/bin/bash
# round-2 GPU session 22: V-row eMA with batched, predicated split-table loads (no term-by-term remainder)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s22_build.log 2>&1
for t in "u17 f32" "u17 f64" "u14-2 f32" "u15-2 f64"; do
  set -- $t
  timeout 900 python bench.py --template $1 --precision $2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/s22_$1_$2.json 2> gpurun_out/s22_$1_$2.err
done
python tools/bsum.py gpurun_out/s22_*.json
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/s22_*.json')):
    try: d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, d.get('ema',{}).get('terms_per_s'), d.get('ema',{}).get('frac_smem'))
    except Exception as e: print(f, e)
PY
timeout 1800 python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py -x -q > gpurun_out/s22_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/s22_tests.log
tail -3 gpurun_out/s22_tests.log
