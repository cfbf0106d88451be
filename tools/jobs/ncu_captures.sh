# round-2 ncu captures: the bench window's resident loop (cfg3, T=20), the cluster sums, the K=64 steady loop
mkdir -p gpurun_out
python tools/profile_window.py cfg3 20 || exit 1
python tools/profile_steady.py k64 300 20 || exit 1
NCU="ncu --set full --clock-control none --import-source on"
timeout 900 $NCU -k regex:lloyd_pass_tc -s 1 -c 1 -o gpurun_out/r02_tc_window_cfg3 -f python tools/profile_window.py cfg3 20 > gpurun_out/r4h_a.log 2>&1
timeout 600 $NCU -k regex:cluster_sums -c 1 -o gpurun_out/r02_sums_cfg3 -f python tools/profile_window.py cfg3 1 > gpurun_out/r4h_b.log 2>&1
timeout 900 $NCU -k regex:lloyd_pass_tc -s 1 -c 1 -o gpurun_out/r02_tc_steady_k64 -f python tools/profile_steady.py k64 300 20 > gpurun_out/r4h_c.log 2>&1
timeout 900 $NCU -k regex:lloyd_pass_tc -s 1 -c 1 -o gpurun_out/r02_tc_steady_cfg3 -f python tools/profile_steady.py cfg3 400 50 > gpurun_out/r4h_d.log 2>&1
ls -la gpurun_out/*.ncu-rep
tail -3 gpurun_out/r4h_*.log
