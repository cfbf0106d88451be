# round 2 (l): peer-exchange resident loop (world 1); shared-atomics microbenchmark
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
(cd tools/ubench && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o atoms atoms.cu && ./atoms) > gpurun_out/r2l_atoms.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_peer.py tests/test_gpu_resident.py -x -q -p no:cacheprovider > gpurun_out/r2l_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/r2l_tests.log
