mkdir -p gpurun_out/r2
for cfg in "GICP_LIN_QUEUE=0 GICP_KNN_ROWS=1" "GICP_LIN_QUEUE=1 GICP_KNN_ROWS=0" "GICP_LIN_QUEUE=0 GICP_KNN_ROWS=0" "GICP_LIN_QUEUE=1 GICP_KNN_ROWS=1"; do
  echo "== $cfg" >> gpurun_out/r2/dbg6.log
  env $cfg timeout 600 python -m pytest tests/test_gpu_batched.py -m gpu -q -p no:cacheprovider >> gpurun_out/r2/dbg6.log 2>&1
done
