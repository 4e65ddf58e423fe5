mkdir -p gpurun_out/r2
timeout 600 python tools/knn_tile_check.py 0.5 > gpurun_out/r2/knn_tile_check5.log 2>&1
timeout 1700 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r2/pytest_gpu_full8.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/r2/smoke8.log 2>&1
timeout 900 python bench.py > gpurun_out/r2/bench_c4_s3c.log 2>&1
timeout 600 python bench.py --workload c3 --no-cpu-baseline > gpurun_out/r2/bench_c3_s3c.log 2>&1
timeout 900 python tools/workloads.py c5 > gpurun_out/r2/workloads_c5_s3c.jsonl 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/r2/bench_launches_s3c.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2/ncu_bench_list_s3c.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_lin_search|k_lin_terms|k_lin_cert" --launch-skip 40 -c 5 -o gpurun_out/r2/prof_lin_bench_s3c python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2/ncu_lin_bench_s3c.log 2>&1
python tools/prof_knn.py 0.5 > /dev/null 2>&1 && ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_knn_tile -c 1 -o gpurun_out/r2/prof_knn_tile_s3c python tools/prof_knn.py 0.5 > gpurun_out/r2/ncu_knn_tile_s3c.log 2>&1
python tools/prof_knn.py 0.5 > /dev/null 2>&1 && ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv python tools/prof_knn.py 0.5 > gpurun_out/r2/knn_launches_s3c.csv 2>&1
