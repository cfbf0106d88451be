# A/B on one box: current library vs the pre-fp64-shadow build (variant pre64), bench cfg3
mkdir -p gpurun_out
for i in 1 2; do
  for v in cur pre64; do
    if [ $v = cur ]; then unset KM_LIB_VARIANT; else export KM_LIB_VARIANT=$v; fi
    python bench.py --steps 20 --warmup 5 > gpurun_out/r4f_$v$i.json 2>/dev/null
    python - <<PY
import json; d = json.load(open("gpurun_out/r4f_$v$i.json"))
print("$v", round(d["ms_per_step"]*1e3, 2), "us/step", "frac", round(d["roofline"]["frac"], 3), "clocks", d["clocks"], d["config"]["timing"])
PY
  done
done
unset KM_LIB_VARIANT
for v in cur pre64; do if [ $v = pre64 ]; then export KM_LIB_VARIANT=pre64; fi; echo $v; python tools/time_steady.py 2>&1 | tail -3; done
