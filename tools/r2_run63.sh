mkdir -p gpurun_out/r2
timeout 600 python tools/prof_c4.py 32 > gpurun_out/r2/prof_c4_32_cthr.log 2>&1
GICP_LIN_COARSE_FIRST=0 timeout 600 python tools/prof_c4.py 32 > gpurun_out/r2/prof_c4_32_cfirst0.log 2>&1
timeout 900 python -m pytest tests/test_gpu_batched.py tests/test_gpu_sharded.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2/pytest_cthr.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2/bench_cthr.log 2>&1
