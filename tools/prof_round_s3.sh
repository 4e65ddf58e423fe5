set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_s3.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_s3.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_s3.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_s3.log 2> gpurun_out/bench_s3.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference_s3.log 2>&1
timeout 300 python tools/prof_step.py > gpurun_out/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_s3.csv python tools/prof_step.py > gpurun_out/ncu_ll.log 2>&1
nvidia-smi > gpurun_out/smi.txt
