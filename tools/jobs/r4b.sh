# A/B: split first pass (default) vs the fused full first pass, whole-call device time
mkdir -p gpurun_out
for v in 0 1; do echo "KM_FULL_FIRST_PASS=$v"; KM_FULL_FIRST_PASS=$v timeout 300 python tools/time_call.py cfg3; done
for v in 0 1; do echo "k64 KM_FULL_FIRST_PASS=$v"; KM_FULL_FIRST_PASS=$v timeout 300 python tools/time_call.py k64; done
