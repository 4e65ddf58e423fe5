"""Search statistics of the batched align (needs the GICP_LIN_PROF=1 variant:
python tools/build_variants.py lprof:-DGICP_LIN_PROF=1, run with
GICP_LIB_VARIANT=.../libgicp_lprof.so). usage: python tools/lin_prof.py [n_distinct]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
import gen
import paper_2308_07173_b200 as g
from paper_2308_07173_b200 import sharding

nd = int(sys.argv[1]) if len(sys.argv) > 1 else 4
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
f = g._lib.gicp_debug_lin_prof
f.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
buf = (ctypes.c_ulonglong * 80)()
f(buf, 1)
T, infos = sharding.align_batched_sharded(g, sd, cs, offsets, imap, cm, T0, plan=plan)
torch.cuda.synchronize()
f(buf, 1)
c = list(buf)
print(f"points evaluated (searching kinds) {c[79]}, cached {c[72]} ({c[72] / max(c[79], 1):.3f})")
print(f"level-0 searches {c[73]}: candidates/search {c[74] / max(c[73], 1):.1f}, voxels/search "
      f"{c[76] / max(c[73], 1):.2f}; warp lockstep slots/warp-call {c[77] / max(c[78], 1):.1f} "
      f"vs useful cands/warp-call {c[74] / max(c[78], 1):.1f} (lanes x)")
print(f"stage 2 (coarser levels) entries {c[1]} ({c[1] / max(c[73], 1):.4f} of searches), "
      f"cands/entry {c[75] / max(c[1], 1):.1f}; ring entries {c[2]}; overflow {c[3]}")
print(f"search cycles/warp mean {c[5] / max(c[0], 1):.0f}, total cycles/warp mean {c[6] / max(c[78], 1):.0f}")
print("search log2 hist", c[8:40])
print(f"certificates {c[64]}: limited by the second-nearest {c[65]}, by a pruned voxel {c[66]}, by the cube {c[67]}")
