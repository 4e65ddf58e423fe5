mkdir -p gpurun_out/r2
timeout 1700 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2/pytest_gpu_final.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/r2/smoke_final.log 2>&1
timeout 900 python bench.py > gpurun_out/r2/bench_c4_final4.log 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2/bench_ref_final4.log 2>&1
timeout 600 python bench.py --workload c3 --no-cpu-baseline > gpurun_out/r2/bench_c3_final4.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/r2/bench_launches_final4.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2/ncu_bench_list_final4.log 2>&1
