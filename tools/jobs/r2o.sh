# round 2 (o): set.le certification; wait-strategy variants; full GPU suite
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2o_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/r2o_tests.log
python tools/time_steady.py cfg3 400 100 > gpurun_out/r2o_steady.txt 2>&1
for v in gw1 es128 es300; do KM_LIB_VARIANT=$v python tools/time_steady.py cfg3 400 100 >> gpurun_out/r2o_steady.txt 2>&1; done
python tools/time_windows.py cfg3 > gpurun_out/r2o_windows.txt 2>&1
python tools/time_call.py cfg3 > gpurun_out/r2o_call.txt 2>&1
