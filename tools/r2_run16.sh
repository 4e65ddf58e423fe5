mkdir -p gpurun_out/r2
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pins.py tests/test_gpu_sharded.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2/pytest_p16.log 2>&1
timeout 900 python tools/workloads.py c5 > gpurun_out/r2/workloads_c5_b.jsonl 2>&1
GICP_DEBUG_STATS=1 timeout 600 python -c "
import sys; sys.path.insert(0, '.')
import numpy as np, torch, gen, paper_2308_07173_b200 as g
mp, q = gen.config_c5()
idx = g.build_index(torch.from_numpy(mp).cuda(), 0.2)
n, d = g.knn(idx, torch.from_numpy(q).cuda(), 32)
torch.cuda.synchronize()
" > gpurun_out/r2/c5_stats.log 2>&1
