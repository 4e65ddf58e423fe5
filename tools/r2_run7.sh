mkdir -p gpurun_out/r2
python tools/knn_sweep.py cells=0.5,0.55,0.6 "envs=GICP_KNN_ROWS=1;GICP_KNN_ROWS=0" > gpurun_out/r2/knn_sweep3.log 2>&1
GICP_KNN_ROWS=1 timeout 600 python tools/knn_tile_check.py 0.55 > gpurun_out/r2/knn_tile_check4.log 2>&1
python tools/debug_sharded.py > gpurun_out/r2/dbg_sharded.log 2>&1
