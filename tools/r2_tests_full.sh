mkdir -p gpurun_out/r2
timeout 1700 python -m pytest tests -m gpu -q -s -x -p no:cacheprovider > gpurun_out/r2/pytest_gpu_full.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r2/bench_after_ldlt.log 2>&1
