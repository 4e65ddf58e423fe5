"""Exercise every kernel of libgicp_b200 once on small inputs, for compute-sanitizer:
  compute-sanitizer --tool memcheck|racecheck|synccheck|initcheck python tools/sanitize_all.py
Each stage prints a line; the sanitizer's summary is the verdict."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import gen
import paper_2308_07173_b200 as g
from paper_2308_07173_b200 import sharding

D = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731


def stage(name):
    torch.cuda.synchronize()
    print("ok", name, flush=True)


src, tgt, T_true, T0 = gen.config_c1(sigma=0.002)
it = g.build_index(D(tgt), 0.5)
isrc = g.build_index(D(src), 0.0)
stage("build_index")
nbr, d2 = g.knn(it, D(src), 10)
g.knn_self(it, 7)
_, _, ct = g.knn_cov_self(it, 10)
_, _, cs = g.knn_cov_self(isrc, 10)
g.knn(it, D(np.array([[5000.0, 0, 0], [np.nan, 0, 0]], np.float32)), 4)   # far + NaN queries
stage("knn / knn_self / knn_cov_self (per-query path)")
# the tiled stage: a dense racetrack section (k = 10 and 20)
mp = gen.racetrack_map(60_000, 5)
sel = np.nonzero(np.abs(mp[:, 0] - 150.0) < 60.0)[0]
dense = np.ascontiguousarray(mp[sel])
idn = g.build_index(D(dense), 1.0)
g.knn_cov_self(idn, 20)
g.knn_cov_self(idn, 10)
q = gen.quantised_cloud(3000, 3, half=3.0)   # exact ties
iq = g.build_index(D(q), 0.5)
g.knn_cov_self(iq, 20)
stage("tiled knn_cov_self (k 20, 10, ties)")
g.covariances(D(tgt), nbr_t := g.knn(it, D(tgt), 10)[0])
g.covariances_kd(D(tgt), nbr_t, "laplacian", sigma=0.5)
g.covariances_kd(D(tgt), nbr_t, "polynomial", alpha=0.01, c=1.0, degree=2, reg="min_eig")
stage("covariances / covariances_kd")
out, corr = g.linearize(D(src), cs, it, ct, T0, 1.0, pivot=T0[:3, 3])
g.linearize(D(src), cs, it, ct, T0, 1.0, corr=corr, reuse_corr=True, error_only=True)
g.attach_cov(it, ct)
g.align(D(src), cs, it, ct, T0)
g.align(D(src), cs, it, ct, T0, lm=False)
stage("linearize / align")
srcs = torch.cat([D(src), D(src)]).contiguous()
covs = torch.cat([cs, cs]).contiguous()
offs = [0, len(src), 2 * len(src)]
g.linearize_batched(srcs, covs, offs, it, ct, np.stack([T0, T_true]))
g.align_batched(srcs, covs, offs, it, ct, np.stack([T0, T0]))
sharding.align_batched_sharded(g, srcs, covs, offs, it, ct, np.stack([T0, T0]))
g.combine_chunks(torch.zeros((2, 8, 32), dtype=torch.float64, device="cuda"), 2, 8, 32)
stage("batched / sharded align, combine_chunks")
iv = g.build_index(D(tgt), 1.0)
g.attach_voxels(iv, ct)
g.linearize_vgicp(D(src), cs, iv, T0, mode=7)
g.align_vgicp(D(src), cs, iv, T0, mode=7)
stage("vgicp")
sc, _ = gen.scan(20_000, 300.0, 78)
g.ground_filter(D(sc), 0.5, 6)
g.cluster(D(sc[:3000]), 0.5, 5)
b = (np.arange(len(mp)) % 50).astype(np.int32)
sm = g.Submap(D(b), 50)
sm.query(3, 2)
sm.free()
stage("ground filter / cluster / submap")
print("ALL STAGES DONE", flush=True)
