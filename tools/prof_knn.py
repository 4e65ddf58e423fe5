"""One C3 map self-kNN+cov call (k=20) after warm-up, for ncu captures:
ncu --profile-from-start off ... python tools/prof_knn.py [cell] [which]
which = map (default) | scan"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import gen
import paper_2308_07173_b200 as g

cell = float(sys.argv[1]) if len(sys.argv) > 1 else 0.5
which = sys.argv[2] if len(sys.argv) > 2 else "map"
sc, mp, T, T0 = gen.config_c3()
pts = mp if which == "map" else sc
idx = g.build_index(torch.from_numpy(np.array(pts)).cuda(), cell if which == "map" else 0.0)
n = len(pts)
out = (torch.empty((n, 20), dtype=torch.int32, device="cuda"), torch.empty((n, 20), dtype=torch.float32, device="cuda"),
       torch.empty((n, 6), dtype=torch.float32, device="cuda"))
for _ in range(3):
    g.knn_cov_self(idx, 20, 1e-3, out=out)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
g.knn_cov_self(idx, 20, 1e-3, out=out)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("done")
