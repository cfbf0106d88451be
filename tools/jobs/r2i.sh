# round 2 (i): change queue offload; steady-state DBG experiments on the tuning build
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_configs.py tests/test_gpu_resident.py tests/test_gpu_tensorcore.py -x -q -p no:cacheprovider > gpurun_out/r2i_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/r2i_tests.log
python tools/time_call.py cfg3 > gpurun_out/r2i_call.txt 2>&1
python tools/time_windows.py cfg3 > gpurun_out/r2i_windows.txt 2>&1
for d in 0 64 68 96 320 192; do KM_LIB_VARIANT=tune KM_TC_DBG=$d python tools/time_steady.py cfg3 400 100 >> gpurun_out/r2i_steady.txt 2>&1; done
python tools/time_steady.py cfg3 400 100 >> gpurun_out/r2i_steady.txt 2>&1
