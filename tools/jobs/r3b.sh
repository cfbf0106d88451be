# round 2 (3b): 4 epilogue groups (K = 64 epilogue-bound?)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
for v in "" epi4; do KM_LIB_VARIANT=$v timeout 300 python tools/time_steady.py k64 250 100 >> gpurun_out/r3b_steady.txt 2>&1; KM_LIB_VARIANT=$v timeout 300 python tools/time_steady.py cfg3 400 100 >> gpurun_out/r3b_steady.txt 2>&1; done
