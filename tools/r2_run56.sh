mkdir -p gpurun_out/r2
for cm in 16384 131072 4194304; do GICP_LIN_COOP_MAX=$cm timeout 600 python tools/prof_c4.py 32 > gpurun_out/r2/prof_c4_32_cm$cm.log 2>&1; done
