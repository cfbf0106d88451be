# round 2 (h): compile-time-m cluster sums; kernel durations of single km_lloyd calls (T=1, T=20)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_configs.py tests/test_gpu_resident.py -x -q -p no:cacheprovider > gpurun_out/r2h_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/r2h_tests.log
python tools/time_call.py cfg3 > gpurun_out/r2h_call.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/r2h_launches_T1.csv python tools/profile_pass.py cfg3 1 > gpurun_out/r2h_ncu1.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/r2h_launches_T20.csv python tools/profile_pass.py cfg3 20 > gpurun_out/r2h_ncu20.log 2>&1
python bench.py --steps 20 --warmup 5 --e2e-steps 1 --cpu-seconds 4 > gpurun_out/r2h_bench.json 2> gpurun_out/r2h_bench.err
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2h_bench_ref.json 2> gpurun_out/r2h_bench_ref.err
