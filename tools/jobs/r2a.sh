# round 2 (a): baseline of HEAD in the driver's window + source-level ncu of the resident pass
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
python bench.py --steps 20 --warmup 5 --skip-cpu --e2e-steps 1 > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err
python tools/time_windows.py cfg3 > gpurun_out/r2a_windows.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:lloyd_pass_tc -s 1 -c 1 -o gpurun_out/r2a_steady python tools/profile_steady.py cfg3 400 20 > gpurun_out/r2a_ncu_steady.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:lloyd_pass_tc -s 1 -c 1 -o gpurun_out/r2a_first python tools/profile_steady.py cfg3 3 20 > gpurun_out/r2a_ncu_first.log 2>&1
