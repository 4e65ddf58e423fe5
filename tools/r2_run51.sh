mkdir -p gpurun_out/r2
python tools/knn_sweep.py cells=0.5 "envs=SCAN_CELL=0;SCAN_CELL=0.35;SCAN_CELL=0.45;SCAN_CELL=0.6;SCAN_CELL=0.8;SCAN_CELL=1.0" > gpurun_out/r2/knn_sweep_scan.log 2>&1
