# round-1 (f): re-verify HEAD after container restore — tests, bench (both arms), launch list, full capture, smoke
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r1f_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/r1f_tests.log
python bench.py > gpurun_out/r1f_bench.json 2> gpurun_out/r1f_bench.err
python bench.py --impl reference > gpurun_out/r1f_bench_ref.json 2> gpurun_out/r1f_bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r1f_launches.csv python bench.py --steps 20 --warmup 3 --skip-e2e --skip-cpu --max-reps 1 > gpurun_out/r1f_ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:lloyd_pass_tc -s 1 -c 1 -o gpurun_out/r1f_tc_full python tools/profile_steady.py cfg3 400 50 > gpurun_out/r1f_ncu_full.log 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r1f_smoke.log 2>&1
