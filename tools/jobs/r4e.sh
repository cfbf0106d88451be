# call overhead: C0 in the begin kernel's parameters, publish kernel instead of 3 D2H copies, lean wrapper
mkdir -p gpurun_out
timeout 300 python tools/time_call.py cfg3
KM_CALL_TRACE=1 timeout 300 python tools/time_call.py cfg2 2>&1 | grep -v trace
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
python bench.py --steps 20 --warmup 5 > gpurun_out/r4e_bench.json 2> gpurun_out/r4e_bench.err; tail -c 600 gpurun_out/r4e_bench.json
