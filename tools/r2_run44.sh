mkdir -p gpurun_out/r2
GICP_DEBUG_SPLIT=1 timeout 600 python tools/prof_c4.py 8 > gpurun_out/r2/split_dbg.log 2>&1
