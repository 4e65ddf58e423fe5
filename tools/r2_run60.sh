mkdir -p gpurun_out/r2
timeout 1200 python -m pytest tests/test_gpu_batched.py tests/test_gpu_parity.py tests/test_gpu_pins.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2/pytest_defer1.log 2>&1
timeout 600 python bench.py --workload c3 --no-cpu-baseline > gpurun_out/r2/bench_c3_defer1.log 2>&1
