mkdir -p gpurun_out/r2
python tools/debug_conv.py > gpurun_out/r2/dbg_conv.log 2>&1
GICP_KNN_ROWS=1 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_knn_tile -c 1 -o gpurun_out/r2/prof_knn_rows python tools/prof_knn.py 0.55 > gpurun_out/r2/ncu_knn_rows.log 2>&1
python tools/prof_c4.py 4 > gpurun_out/r2/prof_c4_plain.log 2>&1
ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_linearize --launch-skip 6 -c 1 -o gpurun_out/r2/prof_lin_c4 python tools/prof_c4.py 4 > gpurun_out/r2/ncu_lin_c4.log 2>&1
timeout 900 python -m pytest tests/test_gpu_sharded.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2/pytest_sharded2.log 2>&1
