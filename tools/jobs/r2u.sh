# round 2 (u): A/B the dynamic tail against the previous kernel (variant "pre"); owner sums fix
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_bench_configs.py tests/test_gpu_resident.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/r2u_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/r2u_tests.log
for rep in 1 2; do
timeout 300 python tools/time_steady.py cfg3 400 100 >> gpurun_out/r2u_steady.txt 2>&1
KM_NO_DYN_TAIL=1 timeout 300 python tools/time_steady.py cfg3 400 100 >> gpurun_out/r2u_steady.txt 2>&1
KM_LIB_VARIANT=pre timeout 300 python tools/time_steady.py cfg3 400 100 >> gpurun_out/r2u_steady.txt 2>&1
done
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:cluster_sums --csv --log-file gpurun_out/r2u_sums.csv python tools/time_first.py 5 > /dev/null 2>&1
