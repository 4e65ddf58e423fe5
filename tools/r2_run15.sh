mkdir -p gpurun_out/r2
timeout 1200 python -m pytest tests/test_gpu_sharded.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2/pytest_sharded_c5.log 2>&1
timeout 900 python tools/workloads.py c5 c2 > gpurun_out/r2/workloads_c5_c2.jsonl 2>&1
