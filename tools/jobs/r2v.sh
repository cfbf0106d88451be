# round 2 (v): back to the static-range kernel (+ time-bounded waits); TMEM ring variants; owner-sums profile
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_bench_configs.py tests/test_gpu_resident.py tests/test_gpu_parity.py tests/test_gpu_peer.py -x -q -p no:cacheprovider > gpurun_out/r2v_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/r2v_tests.log
for v in - ns16 ab6; do KM_LIB_VARIANT=$([ "$v" = "-" ] && echo "" || echo $v) timeout 300 python tools/time_steady.py cfg3 400 100 >> gpurun_out/r2v_steady.txt 2>&1; done
ncu --set full --clock-control none --cache-control none --import-source on -k regex:cluster_sums -s 2 -c 1 -o gpurun_out/r2v_owner python tools/time_first.py 3 > gpurun_out/r2v_ncu.log 2>&1
timeout 300 python tools/time_call.py cfg3 > gpurun_out/r2v_call.txt 2>&1
