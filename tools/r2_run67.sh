mkdir -p gpurun_out/r2
V=$PWD/paper_2308_07173_b200/variants
PROF_SAVE=/tmp/T_new.npy timeout 600 python tools/prof_c4.py 32 > gpurun_out/r2/prof_c4_32_ppt2.log 2>&1
PROF_SAVE=/tmp/T_head.npy GICP_LIB_VARIANT=$V/libgicp_ppt1.so timeout 600 python tools/prof_c4.py 32 > gpurun_out/r2/prof_c4_32_ppt1.log 2>&1
python -c "import numpy as np; a=np.load('/tmp/T_new.npy'); b=np.load('/tmp/T_head.npy'); print('ppt2 vs ppt1 poses bitwise equal:', np.array_equal(a,b), np.abs(a-b).max())" > gpurun_out/r2/ppt_bitwise.log 2>&1
GICP_LIB_VARIANT=$V/libgicp_ppt4.so timeout 600 python tools/prof_c4.py 32 > gpurun_out/r2/prof_c4_32_ppt4.log 2>&1
timeout 900 python -m pytest tests/test_gpu_batched.py tests/test_gpu_sharded.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2/pytest_ppt.log 2>&1
