mkdir -p gpurun_out/r2
timeout 900 python tools/c4_halves.py 32 1,2,4 > gpurun_out/r2/c4_halves.log 2>&1
