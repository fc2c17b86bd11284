for t in u15-1 u14-1 u12-1; do
 for arm in A Y B; do
  unset SG2V_LIB SG2V_TUNE
  [ $arm = Y ] && export SG2V_TUNE=8
  [ $arm = B ] && export SG2V_LIB=ab_old/libsg2v_proj1.so
  timeout 300 python bench.py --template $t --no-cpu-baseline --steps 3 --warmup 2 2>>gpurun_out/r1s18_ab.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$t', '$arm', round(d['value'],4), d['kernel_ms_per_step'].get('step'), d['kernel_ms_per_step'].get('top'), d['clocks']['sm_mhz'])" >> gpurun_out/r1s18_ab.txt
 done
done
