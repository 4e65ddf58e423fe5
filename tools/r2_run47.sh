mkdir -p gpurun_out/r2
timeout 1700 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r2/pytest_gpu_full7.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/r2/smoke7.log 2>&1
timeout 900 python bench.py > gpurun_out/r2/bench_c4_s3b.log 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2/bench_ref_s3b.log 2>&1
