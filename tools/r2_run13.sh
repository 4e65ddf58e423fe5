mkdir -p gpurun_out/r2
ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_linearize --launch-skip 40 -c 1 -o gpurun_out/r2/prof_lin_c4_late python tools/prof_c4.py 8 > gpurun_out/r2/ncu_lin_c4_late.log 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv python tools/prof_c4.py 8 > gpurun_out/r2/lin_c4_launches.csv 2>&1
