"""Sweep of the cube-stage threshold (GICP_LIN_COARSE_THR) on C4: 16 scans x 100k vs
the 2M map, batched and single aligns (ms, median of 3); every setting must give
bitwise the same poses."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import gen
import paper_2308_07173_b200 as g
from tools.workloads import D, timed

B = 16
sc0, mp, _, _ = gen.config_c3()
im = g.build_index(D(mp), 0.5)
_, _, cm = g.knn_cov_self(im, 20, with_nbr=False)
g.attach_cov(im, cm)
scans, covs, T0s = [], [], []
for i in range(B):
    sc, T, T0 = gen.config_c4_scan(i * (256 // B))
    sd = D(sc)
    isc = g.build_index(sd, 0.0)
    _, _, cs = g.knn_cov_self(isc, 20, with_nbr=False)
    isc.free()
    scans.append(sd)
    covs.append(cs)
    T0s.append(T0)
offs = np.concatenate([[0], np.cumsum([s.shape[0] for s in scans])])
src = torch.cat(scans).contiguous()
cov = torch.cat(covs).contiguous()
T0s = np.array(T0s)
ref = None
for thr in sys.argv[1:] or ["inf", "4", "2", "1", "0.4"]:
    os.environ["GICP_LIN_COARSE_THR"] = thr
    ms_b, (Ts, infos) = timed(lambda: g.align_batched(src, cov, offs, im, cm, T0s, allow_degenerate=True), reps=3)
    ms_s, res_s = timed(lambda: [g.align(scans[b], covs[b], im, cm, T0s[b]) for b in range(B)], reps=3)
    Ts = np.asarray(Ts)
    ref = Ts if ref is None else ref
    print(f"thr={thr} batched_ms {ms_b:.2f} singles_ms {ms_s:.2f} same_as_first {np.array_equal(ref, Ts)}", flush=True)
