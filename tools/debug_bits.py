"""Save out29 of a few linearisations (public API, batched API, ERROR_ONLY) to a
file, to compare two builds bit by bit. usage: debug_bits.py out.npy"""
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
res = []
for TT in (T, T0):
    o, c = g.linearize(sd, cs, im, cm, TT, 1.0)
    res.append(o.cpu().numpy())
    o2, _ = g.linearize(sd, cs, im, cm, TT, 1.0, corr=c, reuse_corr=True, error_only=True)
    res.append(o2.cpu().numpy())
np.save(sys.argv[1], np.stack(res))
Ta, ia = g.align(sd, cs, im, cm, T0)
np.save(sys.argv[1].replace(".npy", "_align.npy"), Ta)
print("saved", ia)
