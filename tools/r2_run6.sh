mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_gpu_sharded.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2/pytest_sharded.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2/smoke.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 2 > gpurun_out/r2/bench_c4_a.log 2>&1
python tools/prof_knn.py 0.5 > /dev/null 2>&1 && ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv python tools/prof_knn.py 0.5 > gpurun_out/r2/knn_launches3.csv 2>&1
