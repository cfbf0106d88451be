# round 2 (x): how much does the transform cost? (tuning build: dbg 512 = no transform arithmetic, labels frozen)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
for d in 64 576 68 96 608; do KM_LIB_VARIANT=tune KM_TC_DBG=$d timeout 300 python tools/time_steady.py cfg3 400 100 >> gpurun_out/r2x_steady.txt 2>&1; done
for d in 64 576 96; do KM_LIB_VARIANT=tune KM_TC_DBG=$d timeout 300 python tools/time_steady.py k64 300 50 >> gpurun_out/r2x_steady.txt 2>&1; done
