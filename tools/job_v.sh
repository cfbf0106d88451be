mkdir -p gpurun_out
for c in cfg3 k64 k128; do for v in "" e2; do
  echo "=== $c variant '$v'"
  KM_LIB_VARIANT=$v timeout 120 python tools/time_windows.py $c 2>&1 | tail -n 2
done; done > gpurun_out/v76.log 2>&1
timeout 400 python -m pytest tests -m gpu -x -q > gpurun_out/v76_tests.log 2>&1
