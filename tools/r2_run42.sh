mkdir -p gpurun_out/r2
V=$PWD/paper_2308_07173_b200/variants
PROF_SAVE=/tmp/T_new.npy timeout 600 python tools/prof_c4.py 32 > gpurun_out/r2/prof_c4_32_fpw1.log 2>&1
PROF_SAVE=/tmp/T_head.npy GICP_LIB_VARIANT=$V/libgicp_head5.so timeout 600 python tools/prof_c4.py 32 > gpurun_out/r2/prof_c4_32_head8.log 2>&1
python -c "import numpy as np; a=np.load('/tmp/T_new.npy'); b=np.load('/tmp/T_head.npy'); print('new vs head poses bitwise equal:', np.array_equal(a,b), np.abs(a-b).max())" > gpurun_out/r2/fpw1_bitwise.log 2>&1
timeout 900 python -m pytest tests/test_gpu_batched.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "align or batched or split or cert" > gpurun_out/r2/pytest_fpw1.log 2>&1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv python tools/prof_c4.py 8 > gpurun_out/r2/fpw1_launches.csv 2>&1
for v in fpw4 fpw8; do GICP_LIB_VARIANT=$V/libgicp_$v.so timeout 600 python tools/prof_c4.py 32 > gpurun_out/r2/prof_c4_32_$v.log 2>&1; done
