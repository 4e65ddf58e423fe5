mkdir -p gpurun_out/r2
timeout 1200 python -m pytest tests/test_gpu_batched.py tests/test_gpu_sharded.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2/pytest_batched2.log 2>&1
GICP_DEBUG_ALIGN_HOST=1 python tools/prof_c4.py 32 > gpurun_out/r2/prof_c4_32c.log 2>&1
python tools/l2_bw.py > gpurun_out/r2/l2_bw.json 2>&1
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_all.py > gpurun_out/r2/sanitize_memcheck.log 2>&1
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_all.py > gpurun_out/r2/sanitize_racecheck.log 2>&1
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_all.py > gpurun_out/r2/sanitize_synccheck.log 2>&1
