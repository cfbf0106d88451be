# round 2 (3d): large-K tensor-core pass — parity + cfg4 timing vs the SIMT blocked pass
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r3d_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/r3d_tests.log
timeout 600 python bench.py --config cfg4 --steps 20 --warmup 3 --skip-cpu --e2e-steps 1 --max-reps 5 > gpurun_out/r3d_bench_cfg4.json 2> gpurun_out/r3d_bench_cfg4.err
KM_NO_BIG_K=1 timeout 600 python bench.py --config cfg4 --steps 20 --warmup 3 --skip-cpu --skip-e2e --max-reps 5 > gpurun_out/r3d_bench_cfg4_simt.json 2> gpurun_out/r3d_bench_cfg4_simt.err
