# warp-role split variants: 1 transform group + 4 / 3 epilogue groups vs the product (2 + 3)
mkdir -p gpurun_out
for v in t3e2 t3e3 cur; do
  if [ $v = cur ]; then unset KM_LIB_VARIANT; else export KM_LIB_VARIANT=$v; fi
  python bench.py --steps 20 --warmup 5 > gpurun_out/r4m_$v.json 2>/dev/null
  python -c "import json; d = json.load(open('gpurun_out/r4m_$v.json')); print('$v', round(d['ms_per_step']*1e3, 2), 'us/step', d['clocks']['sm_mhz'])"
  python tools/time_steady.py cfg3 400 50 2>&1 | tail -1
  python tools/time_steady.py k64 150 50 2>&1 | tail -1
done
