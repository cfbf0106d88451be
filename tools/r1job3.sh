set -x
python bench.py > gpurun_out/r1c_bench.json 2> gpurun_out/r1c_bench.err
python bench.py --impl reference > gpurun_out/r1c_bench_ref.json 2> gpurun_out/r1c_bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r1c_launches.csv python bench.py --steps 20 --warmup 3 --skip-e2e --skip-cpu --max-reps 1 > gpurun_out/r1c_ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:lloyd_pass_tc -s 1 -c 1 -o gpurun_out/r1c_tc_full python tools/profile_steady.py cfg3 400 50 > gpurun_out/r1c_ncu_full.log 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r1c_smoke.log 2>&1
