#!/bin/bash
# round-2 GPU session 23: ncu --set full of u15-1's narrow register-gather launches (steps 3 and 4), scale 18
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s23_build.log 2>&1
bash tools/ncu_export.sh s23_s3_u15-1 'astep_kernel<float, double, \(int\)8, ' 0 python tools/prof_one.py u15-1 f32 anchored 1 18
bash tools/ncu_export.sh s23_s4_u15-1 'astep_kernel<float, double, \(int\)32, ' 0 python tools/prof_one.py u15-1 f32 anchored 1 18
du -sh gpurun_out
