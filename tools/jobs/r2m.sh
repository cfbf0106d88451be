# round 2 (m): cluster-sums kernel: full ncu profile, stage-count variant
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:cluster_sums --csv --log-file gpurun_out/r2m_sums4.csv python tools/time_first.py 5 > /dev/null 2>&1
KM_LIB_VARIANT=s8 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:cluster_sums --csv --log-file gpurun_out/r2m_sums8.csv python tools/time_first.py 5 > /dev/null 2>&1
ncu --set full --clock-control none --cache-control none --import-source on -k regex:cluster_sums -s 2 -c 1 -o gpurun_out/r2m_sums python tools/time_first.py 3 > gpurun_out/r2m_ncu.log 2>&1
