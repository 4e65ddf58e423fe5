mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_batched.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2/pytest_conc.log 2>&1
for G in 1 2 4 8; do BENCH_ALIGN_GROUPS=$G timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2/bench_g$G.log 2>&1; done
