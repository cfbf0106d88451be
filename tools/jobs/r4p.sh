# A/B: sparse Δ with paired updates (current) vs per-update chain (variant presparse)
for v in cur presparse cur presparse; do
  if [ $v = cur ]; then unset KM_LIB_VARIANT; else export KM_LIB_VARIANT=$v; fi
  python bench.py --steps 20 --warmup 5 > gpurun_out/r4p_$v.json 2>/dev/null
  python -c "import json; d = json.load(open('gpurun_out/r4p_$v.json')); print('$v', round(d['ms_per_step']*1e3, 2), 'us/step', d['clocks']['sm_mhz'])"
  python tools/time_steady.py k64 150 50 2>&1 | tail -1
done
unset KM_LIB_VARIANT
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | grep -E "AssertionError|passed|failed" | tail -3
