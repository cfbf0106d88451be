# A/B: batched heavy-pass Δ (current) vs per-point chain (variant predrs)
mkdir -p gpurun_out
for v in cur predrs cur predrs; do
  if [ $v = cur ]; then unset KM_LIB_VARIANT; else export KM_LIB_VARIANT=$v; fi
  python bench.py --steps 20 --warmup 5 > gpurun_out/r4n_$v.json 2>/dev/null
  python -c "import json; d = json.load(open('gpurun_out/r4n_$v.json')); print('$v', round(d['ms_per_step']*1e3, 2), 'us/step', d['clocks']['sm_mhz'])"
  python tools/time_call.py cfg3 2>&1 | head -3
done
unset KM_LIB_VARIANT
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
