mkdir -p gpurun_out/r2
timeout 600 python tools/knn_tile_check.py 0.5 > gpurun_out/r2/knn_tile_check2.log 2>&1
python tools/prof_knn.py 0.5 > /dev/null 2>&1 && ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv python tools/prof_knn.py 0.5 > gpurun_out/r2/knn_launches2.csv 2>&1
ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_knn_tile -c 1 -o gpurun_out/r2/prof_knn_tile2 python tools/prof_knn.py 0.5 > gpurun_out/r2/ncu_knn_tile2.log 2>&1
timeout 1700 python -m pytest tests -m gpu -q -s -x -p no:cacheprovider > gpurun_out/r2/pytest_gpu_full2.log 2>&1
