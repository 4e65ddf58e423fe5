"""Sweep of the linearize cube-stage threshold (GICP_LIN_COARSE_THR: level 1 while
the last step moved points more than this) inside gicp_align on C3: total align
time (CUDA events, median of 10), bitwise equality of the poses."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import gen
import paper_2308_07173_b200 as g

sc, mp, T, T0 = gen.config_c3()
md, sd = torch.from_numpy(np.array(mp)).cuda(), torch.from_numpy(np.array(sc)).cuda()
im = g.build_index(md, 0.5)
_, _, cm = g.knn_cov_self(im, 20)
g.attach_cov(im, cm)
isc = g.build_index(sd, 0.0)
_, _, cs = g.knn_cov_self(isc, 20)
res = {}
MODES = sys.argv[1:] or ["inf", "1.0", "0.4", "0.2", "0.1", "0.05", "0.02", "0"]
for mode in MODES:
    os.environ["GICP_LIN_COARSE_THR"] = mode
    for _ in range(3):
        g.align(sd, cs, im, cm, T0)
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        Tm, info = g.align(sd, cs, im, cm, T0)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    res[mode] = Tm
    print(f"thr={mode} align ms median {np.median(ts):.3f} min {np.min(ts):.3f} it {info.iterations}", flush=True)
    print(f"---- thr={mode} host trace", file=sys.stderr, flush=True)
    os.environ["GICP_DEBUG_ALIGN_HOST"] = "1"
    g.align(sd, cs, im, cm, T0)
    torch.cuda.synchronize()
    del os.environ["GICP_DEBUG_ALIGN_HOST"]
print("bitwise equal:", all(np.array_equal(res[MODES[0]], res[m]) for m in MODES))
