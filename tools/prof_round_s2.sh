set -x
python bench.py > gpurun_out/bench_s2.log 2> gpurun_out/bench_s2.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference_s2.log 2>&1
PROF_ONLY= python tools/prof_step.py > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_s2.csv python tools/prof_step.py > gpurun_out/ncu_ll.log 2>&1
PROF_ONLY=knn python tools/prof_step.py > gpurun_out/plain2.log 2>&1 && PROF_ONLY=knn ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_knn -c 3 -o gpurun_out/prof_s2_knn python tools/prof_step.py > gpurun_out/ncu_full.log 2>&1
python tools/prof_step.py > gpurun_out/plain3.log 2>&1 && ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_linearize --launch-skip 10 -c 1 -o gpurun_out/prof_s2_lin python tools/prof_step.py > gpurun_out/ncu_lin.log 2>&1
nvidia-smi > gpurun_out/smi.txt
