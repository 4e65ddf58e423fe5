mkdir -p gpurun_out/r2
V=$PWD/paper_2308_07173_b200/variants
PROF_SAVE=/tmp/T_new.npy timeout 600 python tools/prof_c4.py 32 > gpurun_out/r2/prof_c4_32_lean.log 2>&1
PROF_SAVE=/tmp/T_head.npy GICP_LIB_VARIANT=$V/libgicp_head3.so timeout 600 python tools/prof_c4.py 32 > gpurun_out/r2/prof_c4_32_head6.log 2>&1
python -c "import numpy as np; a=np.load('/tmp/T_new.npy'); b=np.load('/tmp/T_head.npy'); print('new vs head poses bitwise equal:', np.array_equal(a,b), np.abs(a-b).max())" > gpurun_out/r2/lean_bitwise.log 2>&1
for v in lu4 lm5 lu4m5; do GICP_LIB_VARIANT=$V/libgicp_$v.so timeout 600 python tools/prof_c4.py 32 > gpurun_out/r2/prof_c4_32_$v.log 2>&1; done
timeout 900 python -m pytest tests/test_gpu_batched.py tests/test_gpu_sharded.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2/pytest_lean.log 2>&1
