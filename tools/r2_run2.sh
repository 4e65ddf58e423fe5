mkdir -p gpurun_out/r2
python tools/prof_knn.py 0.5 > gpurun_out/r2/prof_knn_plain.log 2>&1 && \
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv python tools/prof_knn.py 0.5 > gpurun_out/r2/knn_launches.csv 2>&1
ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_knn_tile -c 1 -o gpurun_out/r2/prof_knn_tile python tools/prof_knn.py 0.5 > gpurun_out/r2/ncu_knn_tile.log 2>&1
python tools/debug_c3crop3.py > gpurun_out/r2/dbg_c3crop3b.log 2>&1
