# round-1 (e): out-of-line delta update — tests, bench, windows, smoke
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/r1e_tests.log 2>&1 || exit 1
python bench.py > gpurun_out/r1e_bench.json 2> gpurun_out/r1e_bench.err
timeout 120 python tools/time_windows.py cfg3 > gpurun_out/r1e_windows.log 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r1e_smoke.log 2>&1
