mkdir -p gpurun_out/r2
for i in 1 2; do timeout 600 python -m pytest tests/test_gpu_batched.py -m gpu -q -x -p no:cacheprovider -k bitwise_the_single_aligns > gpurun_out/r2/dbg_bt_$i.log 2>&1; done
CUDA_LAUNCH_BLOCKING=1 timeout 600 python -m pytest tests/test_gpu_batched.py -m gpu -q -x -p no:cacheprovider -k bitwise_the_single_aligns > gpurun_out/r2/dbg_bt_blocking.log 2>&1
python tools/debug_batched2.py 64 > gpurun_out/r2/dbg_batched2_64.log 2>&1
