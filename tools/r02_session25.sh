#!/bin/bash
# round-2 GPU session 25: narrow row-group width sized by the gather alone (SG2V_GTDIV) A/B
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s25_build.log 2>&1
for d in 4 16 1000; do
  for t in "u15-1 f32" "u12-1 f32" "u17 f32"; do
    set -- $t
    SG2V_GTDIV=$d timeout 900 python bench.py --template $1 --precision $2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s25_$1_gtdiv$d.json 2> gpurun_out/s25_$1_gtdiv$d.err
  done
  SG2V_GTDIV=$d timeout 900 python bench.py --graph orkut --template u10-2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s25_orkut-u10-2_gtdiv$d.json 2> gpurun_out/s25_orkut-u10-2_gtdiv$d.err
done
python tools/bsum.py gpurun_out/s25_*.json
