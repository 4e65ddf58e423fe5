mkdir -p gpurun_out/r2
GICP_DEBUG_ALIGN_HOST=1 python tools/prof_c4.py 32 > gpurun_out/r2/prof_c4_32.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/r2/bench_c4_b.log 2>&1
