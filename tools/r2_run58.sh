mkdir -p gpurun_out/r2
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv python tools/prof_c4.py 8 > gpurun_out/r2/defer_launches.csv 2>&1
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"k_lin_terms|k_lin_search|k_lin_cert|k_lin_reduce" --launch-skip 80 -c 6 -o gpurun_out/r2/prof_lin_defer python tools/prof_c4.py 8 > gpurun_out/r2/ncu_lin_defer.log 2>&1
