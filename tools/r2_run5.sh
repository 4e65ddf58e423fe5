mkdir -p gpurun_out/r2
python tools/knn_sweep.py cells=0.5,0.55 libs=default > gpurun_out/r2/knn_sweep2.log 2>&1
timeout 600 python tools/knn_tile_check.py 0.5 > gpurun_out/r2/knn_tile_check3.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pins.py tests/test_gpu_sharded.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2/pytest_gpu_p5.log 2>&1
