#!/bin/bash
# round-2 GPU session 27: one-CTA-per-SM bulk gather for wide GENERAL steps (SG2V_BULK1) A/B
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s27_build.log 2>&1
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
for cfg in "u17 f32" "u17 f64" "u16-1 f32" "u17-1 f32"; do
  set -- $cfg
  timeout 900 $B --template $1 --precision $2 > gpurun_out/s27_$1_$2.json 2> gpurun_out/s27_$1_$2.err
  SG2V_BULK1=1 timeout 900 $B --template $1 --precision $2 > gpurun_out/s27_$1_$2_bulk1.json 2> gpurun_out/s27_$1_$2_bulk1.err
done
python tools/bsum.py gpurun_out/s27_*.json
