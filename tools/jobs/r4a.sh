set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fp64_shadow.py -x -q 2>&1 | tail -15
timeout 300 python tools/time_fp64.py 2>&1 | tail -6
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -8
