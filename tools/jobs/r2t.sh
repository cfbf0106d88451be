# round 2 (t): wait-loop variants after the dynamic tail; cluster-owner sums kernel
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_bench_configs.py tests/test_gpu_resident.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/r2t_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/r2t_tests.log
timeout 300 python tools/time_steady.py cfg3 400 100 > gpurun_out/r2t_steady.txt 2>&1
for v in ow h10; do KM_LIB_VARIANT=$v timeout 300 python tools/time_steady.py cfg3 400 100 >> gpurun_out/r2t_steady.txt 2>&1; done
KM_NO_DYN_TAIL=1 timeout 300 python tools/time_steady.py cfg3 400 100 >> gpurun_out/r2t_steady.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:cluster_sums --csv --log-file gpurun_out/r2t_sums.csv python tools/time_first.py 5 > /dev/null 2>&1
timeout 300 python tools/time_call.py cfg3 > gpurun_out/r2t_call.txt 2>&1
