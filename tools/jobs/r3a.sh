# round 2 (3a): per-epilogue-warp private Δ accumulators (no shared atomics)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r3a_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/r3a_tests.log
timeout 300 python tools/time_windows.py cfg3 > gpurun_out/r3a_windows.txt 2>&1
KM_CALL_TRACE=1 timeout 300 python tools/time_call.py cfg3 > gpurun_out/r3a_call.txt 2> gpurun_out/r3a_trace.txt
KM_FULL_FIRST_PASS=1 KM_CALL_TRACE=1 timeout 300 python tools/time_call.py cfg3 > gpurun_out/r3a_call_full.txt 2> gpurun_out/r3a_trace_full.txt
timeout 300 python tools/time_steady.py cfg3 400 100 > gpurun_out/r3a_steady.txt 2>&1
