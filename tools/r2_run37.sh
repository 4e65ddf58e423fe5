mkdir -p gpurun_out/r2
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2/bench_c4_ft.log 2>&1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv python tools/prof_c4.py 8 > gpurun_out/r2/ft_launches.csv 2>&1
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"k_lin_search|k_lin_terms|k_lin_cert" --launch-skip 60 -c 3 -o gpurun_out/r2/prof_lin_ft python tools/prof_c4.py 8 > gpurun_out/r2/ncu_lin_ft.log 2>&1
