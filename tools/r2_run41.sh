mkdir -p gpurun_out/r2
timeout 900 python bench.py > gpurun_out/r2/bench_c4_s3.log 2>&1
timeout 600 python bench.py --workload c3 --no-cpu-baseline > gpurun_out/r2/bench_c3_s3.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/r2/bench_launches_s3.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2/ncu_bench_list_s3.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_lin_search|k_lin_terms|k_lin_cert" --launch-skip 30 -c 4 -o gpurun_out/r2/prof_lin_bench_s3 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2/ncu_lin_bench_s3.log 2>&1
