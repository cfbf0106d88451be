# A/B: cheap retry loop in mbar_wait (current) vs clock per retry (variant mask); cfg3 bench, K=64 windows/steady
mkdir -p gpurun_out
for i in 1 2; do
  for v in cur mask; do
    if [ $v = cur ]; then unset KM_LIB_VARIANT; else export KM_LIB_VARIANT=$v; fi
    python bench.py --steps 20 --warmup 5 > gpurun_out/r4j_$v$i.json 2>/dev/null
    python -c "import json; d = json.load(open('gpurun_out/r4j_$v$i.json')); print('$v', round(d['ms_per_step']*1e3, 2), 'us/step', d['clocks']['sm_mhz'])"
    python tools/time_steady.py cfg3 400 50 2>&1 | tail -1
    python tools/time_steady.py k64 150 50 2>&1 | tail -1
  done
done
