mkdir -p gpurun_out
for v in ni coop e3 ni coop; do echo "=== '$v'"; KM_LIB_VARIANT=$v timeout 120 python tools/time_windows.py cfg3 2>&1; done > gpurun_out/v82.log 2>&1
