# round 2 (k): heavy passes (raw tile released by the epilogue; changed rows from shared memory)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2k_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/r2k_tests.log
python tools/time_steady.py cfg3 400 100 > gpurun_out/r2k_steady.txt 2>&1
python tools/time_windows.py cfg3 > gpurun_out/r2k_windows.txt 2>&1
python tools/time_call.py cfg3 > gpurun_out/r2k_call.txt 2>&1
KM_FULL_FIRST_PASS=1 python tools/time_call.py cfg3 > gpurun_out/r2k_call_full.txt 2>&1
python bench.py --steps 20 --warmup 5 --skip-cpu --e2e-steps 1 > gpurun_out/r2k_bench.json 2> gpurun_out/r2k_bench.err
