#!/bin/bash
# round-2 GPU session 21: the other BASELINE configs at HEAD (Miami-like u5-2/u7-2, Orkut-like u10-2/u12-1, ER u3-1)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s21_build.log 2>&1
for cfg in "miami u5-2" "miami u7-2" "orkut u10-2" "orkut u12-1"; do
  set -- $cfg
  timeout 900 python bench.py --graph $1 --template $2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s21_$1_$2.json 2> gpurun_out/s21_$1_$2.err
  SG2V_WROW=0 timeout 900 python bench.py --graph $1 --template $2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s21_$1_$2_wrow0.json 2> gpurun_out/s21_$1_$2_wrow0.err
done
python tools/bsum.py gpurun_out/s21_*.json
