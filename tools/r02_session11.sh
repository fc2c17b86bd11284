#!/bin/bash
# round-2 GPU session 11: compute-sanitizer memcheck / racecheck / synccheck over every kernel path
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s11_build.log 2>&1
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 2400 $CS --tool memcheck --leak-check no --print-limit 50 python tools/sanitize_run.py > gpurun_out/s11_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/s11_memcheck.log
SG2V_BULK_MIN=1 timeout 2400 $CS --tool memcheck --leak-check no --print-limit 50 python tools/sanitize_run.py > gpurun_out/s11_memcheck_bulk.log 2>&1; echo "memcheck(bulk everywhere) rc=$?" >> gpurun_out/s11_memcheck_bulk.log
timeout 3000 $CS --tool racecheck --racecheck-report analysis --print-limit 50 python tools/sanitize_run.py > gpurun_out/s11_racecheck.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/s11_racecheck.log
timeout 2400 $CS --tool synccheck --print-limit 50 python tools/sanitize_run.py > gpurun_out/s11_synccheck.log 2>&1; echo "synccheck rc=$?" >> gpurun_out/s11_synccheck.log
for f in s11_memcheck s11_memcheck_bulk s11_racecheck s11_synccheck; do echo "== $f"; grep -E "ERROR SUMMARY|sanitize_run|rc=|Error|Race|Hazard" gpurun_out/$f.log | sort | uniq -c | head -12; done
