mkdir -p gpurun_out/r2
timeout 900 python tools/prof_c4_cell.py 8 0.5,0.4,0.35,0.3,0.25,0.7 > gpurun_out/r2/c4_cell_sweep.log 2>&1
