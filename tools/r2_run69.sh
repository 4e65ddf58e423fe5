mkdir -p gpurun_out/r2
V=$PWD/paper_2308_07173_b200/variants
timeout 600 python tools/prof_c4.py 32 > gpurun_out/r2/prof_c4_32_tms4.log 2>&1
for v in tm5 tm6; do GICP_LIB_VARIANT=$V/libgicp_$v.so timeout 600 python tools/prof_c4.py 32 > gpurun_out/r2/prof_c4_32_$v.log 2>&1; done
