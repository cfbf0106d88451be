# A/B on one box after moving the fp64 handling into X64 instantiations
mkdir -p gpurun_out
for i in 1 2; do
  for v in cur pre64; do
    if [ $v = cur ]; then unset KM_LIB_VARIANT; else export KM_LIB_VARIANT=$v; fi
    python bench.py --steps 20 --warmup 5 > gpurun_out/r4g_$v$i.json 2>/dev/null
    python - <<PY
import json; d = json.load(open("gpurun_out/r4g_$v$i.json"))
print("$v", round(d["ms_per_step"]*1e3, 2), "us/step", "frac", round(d["roofline"]["frac"], 3), "clocks", d["clocks"]["sm_mhz"], d["clocks"]["samples"], d["config"]["timing"])
PY
  done
done
unset KM_LIB_VARIANT
timeout 300 python tools/time_steady.py 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_fp64_shadow.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2
timeout 300 python tools/time_fp64.py 2>&1 | tail -4
