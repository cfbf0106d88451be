# round-1 (h): warp-cooperative recheck in the blocked pass + block-parallel repair argmax
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r1p_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/r1p_tests.log
python bench.py --config cfg4 --steps 100 --warmup 3 --max-reps 3 --e2e-steps 1 > gpurun_out/r1p_bench_cfg4.json 2> gpurun_out/r1p_bench_cfg4.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r1p_launches_cfg4.csv python bench.py --config cfg4 --steps 10 --warmup 3 --skip-e2e --skip-cpu --max-reps 1 > gpurun_out/r1p_ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:lloyd_pass_blocked -s 0 -c 1 -o gpurun_out/r1p_blk_full python tools/profile_steady.py cfg4 1 1 > gpurun_out/r1p_ncu.log 2>&1
python bench.py > gpurun_out/r1p_bench.json 2> gpurun_out/r1p_bench.err
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r1p_smoke.log 2>&1
