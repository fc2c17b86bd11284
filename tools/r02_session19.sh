#!/bin/bash
# round-2 GPU session 19: u17 gather-dominated GENERAL step without M_a staging (bulk); ncu of the split eMA launch
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s19_build.log 2>&1
B="python bench.py --template u17 --steps 2 --warmup 3 --no-cpu-baseline"
timeout 900 $B > gpurun_out/s19_u17_f32.json 2> gpurun_out/s19_u17_f32.err
SG2V_UNSTAGE=0 timeout 900 $B > gpurun_out/s19_u17_f32_unstage0.json 2> gpurun_out/s19_u17_f32_unstage0.err
timeout 900 $B --precision f64 > gpurun_out/s19_u17_f64.json 2> gpurun_out/s19_u17_f64.err
python tools/bsum.py gpurun_out/s19_*.json
bash tools/ncu_export.sh s19_ema_u17 "astep_kernel<float, double, 256, 1, [0-9]+, 4, 2>" 4 python tools/prof_one.py u17 f32 anchored 1 18
du -sh gpurun_out
