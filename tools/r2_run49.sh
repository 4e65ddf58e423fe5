mkdir -p gpurun_out/r2
python tools/knn_sweep.py cells=0.5 libs=default,variants/libgicp_t1536m4.so,variants/libgicp_t1024m5.so,variants/libgicp_t1024m6.so,variants/libgicp_t1280m5.so > gpurun_out/r2/knn_sweep_tile.log 2>&1
