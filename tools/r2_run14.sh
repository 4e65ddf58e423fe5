mkdir -p gpurun_out/r2
timeout 1500 python -m pytest tests/test_gpu_batched.py tests/test_gpu_sharded.py tests/test_gpu_parity.py tests/test_gpu_pins.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2/pytest_p14.log 2>&1
GICP_DEBUG_ALIGN_HOST=1 python tools/prof_c4.py 32 > gpurun_out/r2/prof_c4_32e.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/r2/bench_c4_d.log 2>&1
timeout 600 python bench.py --workload c3 --steps 10 --warmup 3 > gpurun_out/r2/bench_c3_d.log 2>&1
