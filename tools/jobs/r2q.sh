# round 2 (q): is the per-CTA pass time systematic (per SM) or random?
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
KM_LIB_VARIANT=tune KM_TC_TIMES=gpurun_out/r2q_tiles.txt python tools/profile_pass.py cfg3 200 > gpurun_out/r2q_tune.log 2>&1
KM_LIB_VARIANT=tune KM_TC_TIMES=gpurun_out/r2q_tiles2.txt python tools/profile_pass.py cfg3 200 >> gpurun_out/r2q_tune.log 2>&1
