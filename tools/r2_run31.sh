mkdir -p gpurun_out/r2
V=$PWD/paper_2308_07173_b200/variants
timeout 600 python tools/prof_c4.py 32 > gpurun_out/r2/prof_c4_32_dyn2.log 2>&1
GICP_LIN_SPLIT_FULL=1 timeout 600 python tools/prof_c4.py 32 > gpurun_out/r2/prof_c4_32_splitfull.log 2>&1
for v in u2m5 u2m6 u4m4; do GICP_LIB_VARIANT=$V/libgicp_$v.so timeout 600 python tools/prof_c4.py 32 > gpurun_out/r2/prof_c4_32_dyn_$v.log 2>&1; done
