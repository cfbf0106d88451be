mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 120 python tools/bigk_repro.py 5000 25 300 > gpurun_out/r3e_a.txt 2>&1
timeout 600 compute-sanitizer --tool memcheck python tools/bigk_repro.py 3000 25 300 > gpurun_out/r3e_memcheck.txt 2>&1
timeout 120 python tools/bigk_repro.py 5000 25 200 > gpurun_out/r3e_b.txt 2>&1
