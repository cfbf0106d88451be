# round 2 (n): register-accumulator cluster sums; per-tile timeline of the resident pass (tuning build)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_bench_configs.py tests/test_gpu_resident.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/r2n_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/r2n_tests.log
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:cluster_sums --csv --log-file gpurun_out/r2n_sums.csv python tools/time_first.py 5 > /dev/null 2>&1
KM_LIB_VARIANT=tune KM_TC_TIMES=gpurun_out/r2n_tiles.txt python tools/profile_pass.py cfg3 150 > gpurun_out/r2n_tune.log 2>&1
python tools/time_call.py cfg3 > gpurun_out/r2n_call.txt 2>&1
