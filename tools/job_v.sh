mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_device.py -x -q > gpurun_out/v85_dev.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/v85_tests.log 2>&1
