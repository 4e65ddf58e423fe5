mkdir -p gpurun_out/r2
timeout 600 python tools/prof_c4.py 32 > gpurun_out/r2/prof_c4_32_coarse_def.log 2>&1
GICP_LIN_COARSE_THR=1e30 timeout 600 python tools/prof_c4.py 32 > gpurun_out/r2/prof_c4_32_coarse_never.log 2>&1
GICP_LIN_COARSE_THR=0.2 timeout 600 python tools/prof_c4.py 32 > gpurun_out/r2/prof_c4_32_coarse_02.log 2>&1
GICP_LIN_COARSE_THR=0.8 timeout 600 python tools/prof_c4.py 32 > gpurun_out/r2/prof_c4_32_coarse_08.log 2>&1
