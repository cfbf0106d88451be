# A/B: cluster sums with paired row updates (current) vs per-row chain (variant presums)
for v in cur presums cur presums; do
  if [ $v = cur ]; then unset KM_LIB_VARIANT; else export KM_LIB_VARIANT=$v; fi
  echo "== $v"; KM_CALL_TRACE=1 python tools/time_first.py 6 2>&1 | tail -1
  KM_CALL_TRACE=1 python tools/time_steady.py k64 150 5 2>&1 | grep trace | tail -1
  python bench.py --steps 20 --warmup 5 > gpurun_out/r4s_$v.json 2>/dev/null
  python -c "import json; d = json.load(open('gpurun_out/r4s_$v.json')); print('$v', round(d['ms_per_step']*1e3, 2), 'us/step', d['clocks']['sm_mhz'])"
done
unset KM_LIB_VARIANT
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | grep -E "AssertionError|passed|failed" | tail -3
