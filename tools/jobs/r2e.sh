# round 2 (e): lean cluster-sums kernel; full GPU suite; per-call timing; launch list
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2e_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/r2e_tests.log
python tools/time_call.py cfg3 > gpurun_out/r2e_call.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2e_launches.csv python tools/profile_pass.py cfg3 20 > gpurun_out/r2e_ncu.log 2>&1
python bench.py --steps 20 --warmup 5 --skip-cpu --e2e-steps 1 > gpurun_out/r2e_bench.json 2> gpurun_out/r2e_bench.err
