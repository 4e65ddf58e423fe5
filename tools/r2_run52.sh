mkdir -p gpurun_out/r2
for w in 2 4 8 16; do BENCH_SCAN_WORKERS=$w timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2/bench_sw$w.log 2>&1; done
