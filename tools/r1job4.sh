# round-1 (d): 3 epilogue groups — tests, windows, bench, launch list, full capture, smoke
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/r1d_tests.log 2>&1 || exit 1
for c in cfg3 k64 k128; do timeout 120 python tools/time_windows.py $c 2>&1 | tail -n 2; done > gpurun_out/r1d_windows.log 2>&1
KM_NO_RESIDENT=1 timeout 120 python tools/time_windows.py cfg3 2>&1 | tail -n 2 >> gpurun_out/r1d_windows.log
python bench.py > gpurun_out/r1d_bench.json 2> gpurun_out/r1d_bench.err
python bench.py --force-sharded --steps 200 --skip-cpu > gpurun_out/r1d_shard.json 2> gpurun_out/r1d_shard.err
python bench.py --impl reference > gpurun_out/r1d_bench_ref.json 2> gpurun_out/r1d_bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r1d_launches.csv python bench.py --steps 20 --warmup 3 --skip-e2e --skip-cpu --max-reps 1 > gpurun_out/r1d_ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:lloyd_pass_tc -s 1 -c 1 -o gpurun_out/r1d_tc_full python tools/profile_steady.py cfg3 400 50 > gpurun_out/r1d_ncu_full.log 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r1d_smoke.log 2>&1
