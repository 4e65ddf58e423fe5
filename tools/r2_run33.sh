mkdir -p gpurun_out/r2
timeout 1700 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r2/pytest_gpu_full5.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/r2/smoke5.log 2>&1
timeout 900 python bench.py --workload c3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2/bench_c3_split.log 2>&1
