set -x
mkdir -p gpurun_out
for i in 1 2; do
BENCH_SCAN_THREAD=0 timeout 600 python bench.py > gpurun_out/ab_thread0_$i.log 2>&1
BENCH_SCAN_THREAD=1 timeout 600 python bench.py > gpurun_out/ab_thread1_$i.log 2>&1
done
