mkdir -p gpurun_out/r2
V=$PWD/paper_2308_07173_b200/variants
PROF_SAVE=/tmp/T_new.npy timeout 600 python tools/prof_c4.py 32 > gpurun_out/r2/prof_c4_32_k64.log 2>&1
PROF_SAVE=/tmp/T_head.npy GICP_LIB_VARIANT=$V/libgicp_head6.so timeout 600 python tools/prof_c4.py 32 > gpurun_out/r2/prof_c4_32_head10.log 2>&1
python -c "import numpy as np; a=np.load('/tmp/T_new.npy'); b=np.load('/tmp/T_head.npy'); print('new vs head poses bitwise equal:', np.array_equal(a,b), np.abs(a-b).max())" > gpurun_out/r2/k64_bitwise.log 2>&1
GICP_LIB_VARIANT=$V/libgicp_lprof.so timeout 600 python tools/lin_prof.py 4 > gpurun_out/r2/lin_prof_cert.log 2>&1
