# round 2 (f): group waits (one polling warp per 4-warp group) + producer-warp cluster sums
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2f_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/r2f_tests.log
python tools/time_call.py cfg3 > gpurun_out/r2f_call.txt 2>&1
python tools/time_windows.py cfg3 > gpurun_out/r2f_windows.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/r2f_launches.csv python tools/profile_pass.py cfg3 20 > gpurun_out/r2f_ncu.log 2>&1
python bench.py --steps 20 --warmup 5 --skip-cpu --e2e-steps 1 > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err
ncu --set full --clock-control none --import-source on -k regex:lloyd_pass_tc -s 1 -c 1 -o gpurun_out/r2f_steady python tools/profile_steady.py cfg3 400 20 > gpurun_out/r2f_ncu_steady.log 2>&1
