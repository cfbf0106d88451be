# round 2 (b): split first pass + lean km_lloyd host path + ADVICE fixes: full GPU suite, windows, bench
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2b_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/r2b_tests.log
python tools/time_windows.py cfg3 > gpurun_out/r2b_windows.txt 2>&1
KM_FULL_FIRST_PASS=1 python tools/time_windows.py cfg3 > gpurun_out/r2b_windows_fullfirst.txt 2>&1
python bench.py --steps 20 --warmup 5 --skip-cpu --e2e-steps 1 > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err
