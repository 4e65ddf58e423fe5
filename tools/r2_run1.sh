mkdir -p gpurun_out/r2
python tools/debug_c3crop4.py > gpurun_out/r2/dbg_c3crop4.log 2>&1
timeout 600 python tools/knn_tile_check.py 0.5 > gpurun_out/r2/knn_tile_check.log 2>&1
