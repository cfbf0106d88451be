# round 2 (g): cluster-sums kernel profile; group wait reverted
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
python tools/time_sums.py cfg3 > gpurun_out/r2g_sums.txt 2>&1
python tools/time_sums.py k64 >> gpurun_out/r2g_sums.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_configs.py -x -q -p no:cacheprovider -k "update or cfg3 or golden" > gpurun_out/r2g_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/r2g_tests.log
ncu --set full --clock-control none --import-source on -k regex:cluster_sums -s 3 -c 1 -o gpurun_out/r2g_sums python tools/time_sums.py cfg3 > gpurun_out/r2g_ncu_sums.log 2>&1
python tools/time_call.py cfg3 > gpurun_out/r2g_call.txt 2>&1
