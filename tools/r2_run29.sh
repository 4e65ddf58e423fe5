mkdir -p gpurun_out/r2
V=$PWD/paper_2308_07173_b200/variants
PROF_SAVE=/tmp/T_new.npy timeout 600 python tools/prof_c4.py 32 > gpurun_out/r2/prof_c4_32_terms.log 2>&1
PROF_SAVE=/tmp/T_head.npy GICP_LIB_VARIANT=$V/libgicp_head.so timeout 600 python tools/prof_c4.py 32 > gpurun_out/r2/prof_c4_32_head2.log 2>&1
python -c "import numpy as np; a=np.load('/tmp/T_new.npy'); b=np.load('/tmp/T_head.npy'); print('new vs head poses bitwise equal:', np.array_equal(a,b), np.abs(a-b).max())" > gpurun_out/r2/terms_bitwise.log 2>&1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv python tools/prof_c4.py 8 > gpurun_out/r2/terms_launches.csv 2>&1
