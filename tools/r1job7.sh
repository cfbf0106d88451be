# round-1 (g): blocked large-K pass — full GPU suite, default bench (cfg3, both arms), cfg4 line, launch list, smoke
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r1n_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/r1n_tests.log
python bench.py > gpurun_out/r1n_bench.json 2> gpurun_out/r1n_bench.err
python bench.py --config cfg4 --steps 100 --warmup 3 --max-reps 3 --e2e-steps 1 > gpurun_out/r1n_bench_cfg4.json 2> gpurun_out/r1n_bench_cfg4.err
python bench.py --impl reference --config cfg4 --steps 2 --warmup 1 > gpurun_out/r1n_bench_cfg4_ref.json 2> gpurun_out/r1n_bench_cfg4_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r1n_launches_cfg4.csv python bench.py --config cfg4 --steps 10 --warmup 3 --skip-e2e --skip-cpu --max-reps 1 > gpurun_out/r1n_ncu_launch.log 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r1n_smoke.log 2>&1
