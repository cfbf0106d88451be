# A/B: candidate mask + popcount (current) vs packed counter chain (variant base); cfg3 bench + K=64 steady
mkdir -p gpurun_out
for i in 1 2; do
  for v in cur base; do
    if [ $v = cur ]; then unset KM_LIB_VARIANT; else export KM_LIB_VARIANT=$v; fi
    python bench.py --steps 20 --warmup 5 > gpurun_out/r4i_$v$i.json 2>/dev/null
    python -c "import json; d = json.load(open('gpurun_out/r4i_$v$i.json')); print('$v', round(d['ms_per_step']*1e3, 2), 'us/step', d['clocks']['sm_mhz'])"
    python tools/time_steady.py k64 2>&1 | tail -1
  done
done
unset KM_LIB_VARIANT
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
