# round 2 (d): bulk-copy cluster sums; per-call timing; launch list; per-phase timing of resident passes (tuning build)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_bench_configs.py tests/test_gpu_resident.py -x -q -p no:cacheprovider > gpurun_out/r2d_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/r2d_tests.log
python tools/time_call.py cfg3 > gpurun_out/r2d_call.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2d_launches.csv python tools/profile_pass.py cfg3 20 > gpurun_out/r2d_ncu.log 2>&1
KM_LIB_VARIANT=tune KM_TC_TIMES=gpurun_out/r2d_phases.txt python tools/profile_pass.py cfg3 200 > gpurun_out/r2d_tune.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:cluster_sums -c 1 -o gpurun_out/r2d_sums python tools/profile_pass.py cfg3 2 > gpurun_out/r2d_ncu_sums.log 2>&1
