# round 2 (w): K3 (one score column per centre) for the shared-memory A path (K = 64: 3 epilogue groups)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2w_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/r2w_tests.log
timeout 300 python tools/time_steady.py k64 400 50 > gpurun_out/r2w_steady.txt 2>&1
KM_LIB_VARIANT=k3off timeout 300 python tools/time_steady.py k64 400 50 >> gpurun_out/r2w_steady.txt 2>&1
timeout 300 python tools/time_steady.py cfg3 400 100 >> gpurun_out/r2w_steady.txt 2>&1
timeout 600 python bench.py --config cfg5 --steps 20 --warmup 3 --skip-cpu --e2e-steps 1 --max-reps 3 > gpurun_out/r2w_bench_cfg5.json 2> gpurun_out/r2w_bench_cfg5.err
