set -x
mkdir -p gpurun_out/r2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2/smi0.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2/pytest_gpu_base.log 2>&1
timeout 300 python tools/kbench.py 10 > gpurun_out/r2/kbench_base.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r2/bench_base.log 2>&1
