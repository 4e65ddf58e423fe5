"""Correspondence-certificate statistics of gicp_align on C3 (GICP_DEBUG_ALIGN=1):
per iteration the valid certificates, how many were carried from the previous
iteration without a search, rho percentiles; plus the host trace (per launch wait)
with and without the certificates."""
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
for _ in range(3):
    g.align(sd, cs, im, cm, T0)
torch.cuda.synchronize()
for mode in ("cache", "nocache"):
    if mode == "nocache":
        os.environ["GICP_ALIGN_NOCACHE"] = "1"
    print(f"---- {mode}: stats", file=sys.stderr, flush=True)
    os.environ["GICP_DEBUG_ALIGN"] = "1"
    g.align(sd, cs, im, cm, T0)
    torch.cuda.synchronize()
    del os.environ["GICP_DEBUG_ALIGN"]
    print(f"---- {mode}: host trace", file=sys.stderr, flush=True)
    os.environ["GICP_DEBUG_ALIGN_HOST"] = "1"
    g.align(sd, cs, im, cm, T0)
    torch.cuda.synchronize()
    del os.environ["GICP_DEBUG_ALIGN_HOST"]
