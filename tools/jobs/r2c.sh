# round 2 (c): per-call timing + launch list of one 20-iteration km_lloyd call
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
python tools/time_call.py cfg3 > gpurun_out/r2c_call.txt 2>&1
KM_FULL_FIRST_PASS=1 python tools/time_call.py cfg3 > gpurun_out/r2c_call_fullfirst.txt 2>&1
python tools/time_windows.py cfg3 > gpurun_out/r2c_windows.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2c_launches.csv python tools/profile_pass.py cfg3 20 > gpurun_out/r2c_ncu.log 2>&1
