# round 2 (y): per-step device/host trace of km_lloyd calls
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
KM_CALL_TRACE=1 timeout 300 python tools/time_call.py cfg3 > gpurun_out/r2y_call.txt 2> gpurun_out/r2y_trace.txt
