set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_s3b.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_s3b.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_s3b.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_s3b.log 2> gpurun_out/bench_s3b.err
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e > gpurun_out/bench_s3b_short.log 2>&1
nvidia-smi > gpurun_out/smi.txt
