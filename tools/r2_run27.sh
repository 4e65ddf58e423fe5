mkdir -p gpurun_out/r2
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"k_linearize|k_lin_cert" --launch-skip 60 -c 3 -o gpurun_out/r2/prof_lin_s13 python tools/prof_c4.py 8 > gpurun_out/r2/ncu_lin_s13.log 2>&1
