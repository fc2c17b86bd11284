#!/bin/bash
# Full-size oracle goldens for the bench workload (u15-1 on RMAT-1M-like), run on the
# GPU box's host cores (196 GB RAM; the oracle's peak at root 0 is ~109 GB).
mkdir -p gpurun_out
bash tools/hostinfo.sh
python -c "from oracle import oracle as O; O.build()"
timeout 7000 python tools/make_golden_big.py --case rmat1m:u15-1:0:u64,f64 --case rmat1m:u15-1:5:u64 \
    --rows 4096 --out gpurun_out/golden_u15.json > gpurun_out/golden_u15.log 2>&1
echo "rc=$?" >> gpurun_out/golden_u15.log
tail -c 3000 gpurun_out/golden_u15.log
