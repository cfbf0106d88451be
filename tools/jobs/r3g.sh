mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python tools/time_fp64.py > gpurun_out/r3g_fp64.txt 2>&1
