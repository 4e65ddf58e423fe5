mkdir -p gpurun_out/r2
V=$PWD/paper_2308_07173_b200/variants
python tools/knn_sweep.py cells=0.5 libs=default,variants/libgicp_head3.so > gpurun_out/r2/knn_sweep_ring2.log 2>&1
python tools/prof_knn.py 0.5 > /dev/null 2>&1 && ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv python tools/prof_knn.py 0.5 > gpurun_out/r2/knn_launches_ring2.csv 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pins.py tests/test_gpu_sharded.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2/pytest_ring2.log 2>&1
timeout 900 python tools/workloads.py c5 > gpurun_out/r2/workloads_c5_ring2.jsonl 2>&1
