mkdir -p gpurun_out/r2
python tools/knn_sweep.py cells=0.45,0.5,0.55 libs=default,variants/libgicp_minb5.so > gpurun_out/r2/knn_sweep1.log 2>&1
