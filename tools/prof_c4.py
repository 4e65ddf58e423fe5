"""A reduced C4 batch (N distinct scans x 8 hypotheses) aligned once through
gicp_align_batched_sharded, the align inside cudaProfilerStart/Stop (ncu
--profile-from-start off -k regex:k_linearize --launch-skip S -c 1).
usage: python tools/prof_c4.py [n_distinct]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
import gen
import paper_2308_07173_b200 as g
from paper_2308_07173_b200 import sharding

nd = int(sys.argv[1]) if len(sys.argv) > 1 else 8
scans = bench.gen_scans(list(range(nd)), min(nd, os.cpu_count() or 1))
mp = gen.racetrack_map(2_000_000, 1)
dev = torch.device("cuda:0")
md = torch.from_numpy(mp).to(dev)
sd = torch.from_numpy(np.concatenate([s for s, _ in scans])).to(dev)
imap = g.build_index(md, bench.MAP_CELL)
_, _, cm = g.knn_cov_self(imap, 20, 1e-3)
g.attach_cov(imap, cm)
cs = torch.empty((nd * bench.N_SCAN, 6), dtype=torch.float32, device=dev)
for i in range(nd):
    isc = g.build_index(sd[i * bench.N_SCAN:(i + 1) * bench.N_SCAN], 0.0)
    g.knn_cov_self(isc, 20, 1e-3, out=(None, None, cs[i * bench.N_SCAN:(i + 1) * bench.N_SCAN]))
B = nd * bench.N_HYP
_, T0 = bench.c4_poses()
T0 = T0[:B]
offsets = np.arange(B + 1, dtype=np.int64) * bench.N_SCAN
plan = sharding.ShardPlan(offsets, dev, reg_base=(np.arange(B) // bench.N_HYP) * bench.N_SCAN)
sharding.align_batched_sharded(g, sd, cs, offsets, imap, cm, T0, plan=plan)   # warm-up
torch.cuda.synchronize()
g.align_timing(True)
torch.cuda.cudart().cudaProfilerStart()
T, infos = sharding.align_batched_sharded(g, sd, cs, offsets, imap, cm, T0, plan=plan)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
ms, n, pts = g.align_timing(False)
print("iterations", [i.iterations for i in infos][:16], "launch ms", ms, "n", n, "pts", pts)
for k in range(3):
    if n[k]:
        print(f"kind {k}: {ms[k] / n[k]:.3f} ms/launch, {pts[k] / n[k]:.0f} pts/launch, "
              f"{80 * pts[k] / (ms[k] * 1e-3) / 1e9:.1f} GB/s")
