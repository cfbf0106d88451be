# round 2 (j): A = [xh|xl] (no third copy), FADD2 transform; 3-transform-group variant
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_tensorcore.py tests/test_gpu_parity.py tests/test_gpu_bench_configs.py -x -q -p no:cacheprovider > gpurun_out/r2j_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/r2j_tests.log
python tools/time_steady.py cfg3 400 100 > gpurun_out/r2j_steady.txt 2>&1
KM_LIB_VARIANT=tg3 python tools/time_steady.py cfg3 400 100 >> gpurun_out/r2j_steady.txt 2>&1
python tools/time_windows.py cfg3 > gpurun_out/r2j_windows.txt 2>&1
KM_LIB_VARIANT=tg3 python tools/time_windows.py cfg3 > gpurun_out/r2j_windows_tg3.txt 2>&1
python tools/time_call.py cfg3 > gpurun_out/r2j_call.txt 2>&1
KM_LIB_VARIANT=tg3 python tools/time_call.py cfg3 > gpurun_out/r2j_call_tg3.txt 2>&1
