mkdir -p gpurun_out/r2
V=$PWD/paper_2308_07173_b200/variants
PROF_SAVE=/tmp/T_new.npy timeout 600 python tools/prof_c4.py 32 > gpurun_out/r2/prof_c4_32_ft.log 2>&1
PROF_SAVE=/tmp/T_head.npy GICP_LIB_VARIANT=$V/libgicp_head2.so timeout 600 python tools/prof_c4.py 32 > gpurun_out/r2/prof_c4_32_head5.log 2>&1
python -c "import numpy as np; a=np.load('/tmp/T_new.npy'); b=np.load('/tmp/T_head.npy'); print('new vs head poses bitwise equal:', np.array_equal(a,b), np.abs(a-b).max())" > gpurun_out/r2/ft_bitwise.log 2>&1
for v in lb5 lb6; do GICP_LIB_VARIANT=$V/libgicp_$v.so timeout 600 python tools/prof_c4.py 32 > gpurun_out/r2/prof_c4_32_$v.log 2>&1; done
timeout 1700 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r2/pytest_gpu_full6.log 2>&1
timeout 900 python bench.py --workload c3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2/bench_c3_ft.log 2>&1
