"""Linearize diagnostics on C3 (needs a GICP_LIN_PROF=1 build + GICP_DEBUG_STATS=1):
one linearize at T_true and one at T0, per-warp search/total cycle histograms."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import gen
import paper_2308_07173_b200 as g

sc, mp, T, T0 = gen.config_c3()
md = torch.from_numpy(np.array(mp)).cuda()
sd = torch.from_numpy(np.array(sc)).cuda()
im = g.build_index(md, 0.5)
_, _, cm = g.knn_cov_self(im, 20, 1e-3)
g.attach_cov(im, cm)
isc = g.build_index(sd, 0.0)
_, _, cs = g.knn_cov_self(isc, 20, 1e-3)
torch.cuda.synchronize()
for name, TT in (("T_true", T), ("T0", T0)):
    for r in range(3):
        print(name, flush=True)
        g.linearize(sd, cs, im, cm, TT, 1.0)
        torch.cuda.synchronize()
