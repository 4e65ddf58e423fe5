mkdir -p gpurun_out/r2
python tools/knn_sweep.py cells=0.5 libs=default,variants/libgicp_es2.so,variants/libgicp_es4.so,variants/libgicp_es9.so > gpurun_out/r2/knn_sweep_esc.log 2>&1
