# round 2 (s): dynamic tail (pool tiles + sentinels through the rings); time-bounded mbarrier waits
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2s_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/r2s_tests.log
timeout 300 python tools/time_steady.py cfg3 400 100 > gpurun_out/r2s_steady.txt 2>&1
KM_NO_DYN_TAIL=1 timeout 300 python tools/time_steady.py cfg3 400 100 >> gpurun_out/r2s_steady.txt 2>&1
timeout 300 python tools/time_windows.py cfg3 > gpurun_out/r2s_windows.txt 2>&1
timeout 300 python tools/time_call.py cfg3 > gpurun_out/r2s_call.txt 2>&1
KM_NO_DYN_TAIL=1 timeout 300 python tools/time_call.py cfg3 > gpurun_out/r2s_call_static.txt 2>&1
