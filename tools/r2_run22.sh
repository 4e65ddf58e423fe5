mkdir -p gpurun_out/r2
V=$PWD/paper_2308_07173_b200/variants
PROF_SAVE=/tmp/T_split.npy timeout 600 python tools/prof_c4.py 32 > gpurun_out/r2/prof_c4_32_split.log 2>&1
PROF_SAVE=/tmp/T_fused.npy GICP_LIN_FUSED=1 timeout 600 python tools/prof_c4.py 32 > gpurun_out/r2/prof_c4_32_fused.log 2>&1
python -c "import numpy as np; a=np.load('/tmp/T_split.npy'); b=np.load('/tmp/T_fused.npy'); print('split vs fused poses bitwise equal:', np.array_equal(a,b), np.abs(a-b).max())" > gpurun_out/r2/split_bitwise.log 2>&1
for v in sminb4 sminb5 sminb8; do GICP_LIB_VARIANT=$V/libgicp_$v.so timeout 600 python tools/prof_c4.py 32 > gpurun_out/r2/prof_c4_32_$v.log 2>&1; done
timeout 1200 python -m pytest tests/test_gpu_batched.py tests/test_gpu_parity.py tests/test_gpu_pins.py tests/test_gpu_sharded.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2/pytest_split.log 2>&1
