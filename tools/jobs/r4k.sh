# epilogue wait back-off variants + stage attribution (tuning build: DBG 4 stream only, 32 no epilogue work)
mkdir -p gpurun_out
for v in cur epi64 epi200; do
  if [ $v = cur ]; then unset KM_LIB_VARIANT; else export KM_LIB_VARIANT=$v; fi
  python bench.py --steps 20 --warmup 5 > gpurun_out/r4k_$v.json 2>/dev/null
  python -c "import json; d = json.load(open('gpurun_out/r4k_$v.json')); print('$v', round(d['ms_per_step']*1e3, 2), 'us/step', d['clocks']['sm_mhz'])"
  python tools/time_steady.py cfg3 400 50 2>&1 | tail -1
  python tools/time_steady.py k64 150 50 2>&1 | tail -1
done
export KM_LIB_VARIANT=tune
for d in 0 4 32; do
  KM_TC_DBG=$d python tools/time_steady.py cfg3 400 50 2>&1 | tail -1
  KM_TC_DBG=$d python tools/time_steady.py k64 150 50 2>&1 | tail -1
done
