mkdir -p gpurun_out/r2
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2/bench_overlap.log 2>&1
