"""Time the fused kNN+covariance on the C3 map (and the scan) for A/B of builds.
usage: GICP_LIB_VARIANT=path.so python tools/kbench.py [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import gen
import paper_2308_07173_b200 as g

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
sc, mp, T, T0 = gen.config_c3()
md = torch.from_numpy(np.array(mp)).cuda()
sd = torch.from_numpy(np.array(sc)).cuda()
im = g.build_index(md, float(os.environ.get("KB_CELL", "0.5")))
isc = g.build_index(sd, 0.0)
out = (torch.empty((mp.shape[0], 20), dtype=torch.int32, device="cuda"),
       torch.empty((mp.shape[0], 20), dtype=torch.float32, device="cuda"),
       torch.empty((mp.shape[0], 6), dtype=torch.float32, device="cuda"))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for name, idx, o in (("map", im, out), ("scan", isc, None)):
    ts = []
    for r in range(reps + 2):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.knn_cov_self(idx, 20, 1e-3, out=o)
        b.record()
        torch.cuda.synchronize()
        if r >= 2:
            ts.append(a.elapsed_time(b))
    print(f"{os.path.basename(os.environ.get('GICP_LIB_VARIANT', 'default'))} {name} knn_cov ms median {np.median(ts):.3f} min {np.min(ts):.3f}")
