# round 2 (r): one gpu-scope fence per CTA at the grid barrier; certification loop back to FSETP+add
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_resident.py tests/test_gpu_parity.py tests/test_gpu_bench_configs.py tests/test_gpu_peer.py -x -q -p no:cacheprovider > gpurun_out/r2r_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/r2r_tests.log
python tools/time_steady.py cfg3 400 100 > gpurun_out/r2r_steady.txt 2>&1
python tools/time_call.py cfg3 > gpurun_out/r2r_call.txt 2>&1
