mkdir -p gpurun_out/r2
V=$PWD/paper_2308_07173_b200/variants
GICP_LIB_VARIANT=$V/libgicp_lprof.so timeout 600 python tools/lin_prof.py 4 > gpurun_out/r2/lin_prof_base.log 2>&1
