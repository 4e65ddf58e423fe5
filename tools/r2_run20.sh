mkdir -p gpurun_out/r2
V=$PWD/paper_2308_07173_b200/variants
GICP_LIB_VARIANT=$V/libgicp_lprof.so timeout 600 python tools/lin_prof.py 4 > gpurun_out/r2/lin_prof_base.log 2>&1
GICP_LIB_VARIANT=$V/libgicp_lprofwarm.so timeout 600 python tools/lin_prof.py 4 > gpurun_out/r2/lin_prof_warm.log 2>&1
PROF_SAVE=/tmp/T_base.npy timeout 600 python tools/prof_c4.py 32 > gpurun_out/r2/prof_c4_32_base2.log 2>&1
PROF_SAVE=/tmp/T_warm.npy GICP_LIB_VARIANT=$V/libgicp_warm.so timeout 600 python tools/prof_c4.py 32 > gpurun_out/r2/prof_c4_32_warm.log 2>&1
python -c "import numpy as np; a=np.load('/tmp/T_base.npy'); b=np.load('/tmp/T_warm.npy'); print('warm vs base poses bitwise equal:', np.array_equal(a,b), np.abs(a-b).max())" > gpurun_out/r2/warm_bitwise.log 2>&1
GICP_LIB_VARIANT=$V/libgicp_warm.so timeout 900 python -m pytest tests/test_gpu_batched.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "align or batched or lin" > gpurun_out/r2/pytest_warm.log 2>&1
