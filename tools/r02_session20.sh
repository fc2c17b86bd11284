#!/bin/bash
# round-2 GPU session 20: ncu --set full of the split eMA launch (u17 10 = 5 + 5) and of u17's 16 = 10 + 6 step, scale 18
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s20_build.log 2>&1
bash tools/ncu_export.sh s20_ema_u17 'astep_kernel.*\(int\)4, \(int\)2>' 4 python tools/prof_one.py u17 f32 anchored 1 18
bash tools/ncu_export.sh s20_ema_u17_f64 'astep_kernel.*\(int\)2, \(int\)2>' 4 python tools/prof_one.py u17 f64 anchored 1 18
du -sh gpurun_out
