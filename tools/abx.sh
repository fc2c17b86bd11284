#!/bin/bash
# A/B of launch-configuration knobs on one box: tools/abx.sh <tag> <templates...>
# arms: D = default, W16 = SG2V_TUNE=16 (wide rows U=16), P = anchored_plain, B = $LIBB
tag=$1; shift
for t in "$@"; do
 for arm in ${ARMS:-D W16 P}; do
  unset SG2V_LIB SG2V_TUNE; lay=anchored
  [ $arm = W16 ] && export SG2V_TUNE=16
  [ $arm = P ] && lay=anchored_plain
  [ $arm = B ] && export SG2V_LIB=$LIBB
  case $arm in V*) export SG2V_VTPB=${arm#V};; *) unset SG2V_VTPB;; esac
  unset SG2V_HINT; case $arm in H0*) export SG2V_HINT=0;; esac
  unset SG2V_HOTFRAC; case $arm in F*) export SG2V_HOTFRAC=${arm#F};; esac
  case $arm in *P) lay=anchored_plain;; esac
  timeout 300 python bench.py --template $t --layout $lay --no-cpu-baseline --steps 3 --warmup 2 2>>gpurun_out/${tag}_ab.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$t', '$arm', round(d['value'],4), d['kernel_ms_per_step'].get('step'), d['kernel_ms_per_step'].get('top'), d['clocks']['sm_mhz'], d['config']['workspace_GB'])" >> gpurun_out/${tag}_ab.txt
 done
done
