mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_gpu_batched.py tests/test_gpu_sharded.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2/pytest_split7.log 2>&1
timeout 900 python bench.py --workload c3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2/bench_c3_split2.log 2>&1
timeout 600 python tools/prof_c4.py 32 > gpurun_out/r2/prof_c4_32_split7.log 2>&1
