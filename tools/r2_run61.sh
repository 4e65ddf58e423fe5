mkdir -p gpurun_out/r2
timeout 1700 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2/pytest_gpu_final.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/r2/smoke_final.log 2>&1
timeout 900 python bench.py > gpurun_out/r2/bench_c4_final3.log 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2/bench_ref_final3.log 2>&1
timeout 600 python bench.py --workload c3 --no-cpu-baseline > gpurun_out/r2/bench_c3_final3.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/r2/bench_launches_final3.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2/ncu_bench_list_final3.log 2>&1
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"k_lin_terms|k_lin_search|k_lin_cert|k_lin_reduce" --launch-skip 80 -c 6 -o gpurun_out/r2/prof_lin_final3 python tools/prof_c4.py 8 > gpurun_out/r2/ncu_lin_final3.log 2>&1
