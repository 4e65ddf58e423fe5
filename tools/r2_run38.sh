mkdir -p gpurun_out/r2
V=$PWD/paper_2308_07173_b200/variants
timeout 600 python tools/prof_c4.py 32 > gpurun_out/r2/prof_c4_32_base8.log 2>&1
GICP_LIB_VARIANT=$V/libgicp_stream.so timeout 600 python tools/prof_c4.py 32 > gpurun_out/r2/prof_c4_32_stream.log 2>&1
GICP_L2_PERSIST=64 timeout 600 python tools/prof_c4.py 32 > gpurun_out/r2/prof_c4_32_persist.log 2>&1
GICP_L2_PERSIST=64 GICP_LIB_VARIANT=$V/libgicp_stream.so timeout 600 python tools/prof_c4.py 32 > gpurun_out/r2/prof_c4_32_persist_stream.log 2>&1
