mkdir -p gpurun_out/r2
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv python tools/prof_c4.py 8 > gpurun_out/r2/agg_launches.csv 2>&1
