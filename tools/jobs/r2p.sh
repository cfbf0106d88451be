# round 2 (p): full ncu capture of the steady resident loop (current code)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
ncu --set full --clock-control none --import-source on -k regex:lloyd_pass_tc -s 3 -c 1 -o gpurun_out/r2p_steady python tools/profile_steady.py cfg3 400 20 > gpurun_out/r2p_ncu.log 2>&1
