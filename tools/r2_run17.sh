mkdir -p gpurun_out/r2
python tools/debug_ext.py > gpurun_out/r2/dbg_ext3.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pins.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2/pytest_p17.log 2>&1
timeout 900 python tools/workloads.py c5 > gpurun_out/r2/workloads_c5_c.jsonl 2>&1
GICP_LIB_VARIANT=$PWD/paper_2308_07173_b200/variants/libgicp_flat.so timeout 900 python -m pytest tests/test_gpu_batched.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2/pytest_flat.log 2>&1
GICP_DEBUG_ALIGN_HOST=1 python tools/prof_c4.py 32 > gpurun_out/r2/prof_c4_32_base.log 2>&1
GICP_LIB_VARIANT=$PWD/paper_2308_07173_b200/variants/libgicp_flat.so GICP_DEBUG_ALIGN_HOST=1 python tools/prof_c4.py 32 > gpurun_out/r2/prof_c4_32_flat.log 2>&1
