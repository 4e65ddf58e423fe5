mkdir -p gpurun_out/r2
timeout 1200 python -m pytest tests/test_gpu_batched.py tests/test_gpu_sharded.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2/pytest_batched.log 2>&1
GICP_DEBUG_ALIGN_HOST=1 python tools/prof_c4.py 32 > gpurun_out/r2/prof_c4_32b.log 2>&1
