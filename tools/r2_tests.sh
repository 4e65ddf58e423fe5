set -x
mkdir -p gpurun_out/r2
timeout 1500 python -m pytest tests/test_gpu_pins.py tests/test_gpu_parity.py tests/test_gpu_ground.py -m gpu -q -s -x > gpurun_out/r2/pytest_pins.log 2>&1
