set -x
mkdir -p gpurun_out
timeout 300 python tools/prof_step.py > gpurun_out/plain3.log 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_linearize --launch-skip 10 -c 1 -o gpurun_out/prof_s3_lin python tools/prof_step.py > gpurun_out/ncu_lin_s3.log 2>&1
PROF_ONLY=knn timeout 300 python tools/prof_step.py > gpurun_out/plain2.log 2>&1 && PROF_ONLY=knn timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_knn_level -c 1 -o gpurun_out/prof_s3_knn python tools/prof_step.py > gpurun_out/ncu_knn_s3.log 2>&1
