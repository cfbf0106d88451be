# round-2 ncu captures of the final kernels: the bench window's resident loop (cfg3, T=20), a long
# resident run at cfg3 and at K = 64, the cluster sums.  Reports stay in /tmp on the box (gpurun
# copies back at most 64 MiB); their raw-page summaries and the window report come back.
mkdir -p gpurun_out/ncu /tmp/ncu
python tools/profile_window.py cfg3 20 || exit 1
python tools/profile_steady.py k64 300 20 || exit 1
NCU="ncu --set full --clock-control none --import-source on"
timeout 900 $NCU -k regex:lloyd_pass_tc -s 1 -c 1 -o /tmp/ncu/r02_tc_window_cfg3 -f python tools/profile_window.py cfg3 20 > gpurun_out/ncu/a.log 2>&1
timeout 600 $NCU -k regex:cluster_sums -c 1 -o /tmp/ncu/r02_sums_cfg3 -f python tools/profile_window.py cfg3 1 > gpurun_out/ncu/b.log 2>&1
timeout 900 $NCU -k regex:lloyd_pass_tc -s 1 -c 1 -o /tmp/ncu/r02_tc_steady_k64 -f python tools/profile_steady.py k64 300 20 > gpurun_out/ncu/c.log 2>&1
timeout 900 $NCU -k regex:lloyd_pass_tc -s 1 -c 1 -o /tmp/ncu/r02_tc_steady_cfg3 -f python tools/profile_steady.py cfg3 400 50 > gpurun_out/ncu/d.log 2>&1
for r in r02_tc_window_cfg3 r02_sums_cfg3 r02_tc_steady_k64 r02_tc_steady_cfg3; do
  ncu -i /tmp/ncu/$r.ncu-rep --page raw --csv > gpurun_out/ncu/$r.raw.csv 2>/dev/null
done
cp /tmp/ncu/r02_tc_window_cfg3.ncu-rep gpurun_out/ncu/
ls -la /tmp/ncu gpurun_out/ncu
