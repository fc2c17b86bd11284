#!/bin/bash
# A/B timing of library builds / layouts on the same box (bench.py lines, no CPU baseline):
#   tools/ab.sh <tag> <lib_b> <templates...>
# arms: A = in-tree build (default layout), P = in-tree "anchored_plain", B = SG2V_LIB=<lib_b>
tag=$1; libb=$2; shift 2
ARMS=${ARMS:-"A P B A"}
for t in "$@"; do
  for arm in $ARMS; do
    lay=anchored; unset SG2V_LIB
    [ $arm = P ] && lay=anchored_plain
    [ $arm = B ] && export SG2V_LIB=$libb
    timeout 300 python bench.py --template $t --layout $lay --no-cpu-baseline --steps 3 --warmup 2 2>>gpurun_out/${tag}_ab.err | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$t', '$arm', round(d['value'],4), d['kernel_ms_per_step'].get('step'), d['kernel_ms_per_step'].get('top'), d['clocks']['sm_mhz'], d['config'].get('workspace_GB'))" >> gpurun_out/${tag}_ab.txt
  done
done
