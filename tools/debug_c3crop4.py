"""C3 cropped fixture: the align's first linearisation (GICP_DEBUG_ALIGN) vs the public
gicp_linearize at T0 with the same pivot; and a shifted C1 GN step vs the oracle."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import gen
import oracle
import paper_2308_07173_b200 as g
from tests.test_gpu_pins import _c3_cropped

D = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
np.set_printoptions(precision=9, suppress=False, linewidth=200)
# shifted C1: both clouds +300 m in x, T0 = translation (300,...) composition
src, tgt, T_true, T0 = gen.config_c1(sigma=0.002)
S = gen.make_T(np.eye(3), [300.0, -200.0, 5.0])
tgt_s = gen.apply_T(S, tgt).astype(np.float32)
T0s = S @ T0
nt, _ = oracle.knn(tgt_s, tgt_s, 10)
ns, _ = oracle.knn(src, src, 10)
ct = oracle.covariance(tgt_s, nt)[0].astype(np.float32)
cs = oracle.covariance(src, ns)[0].astype(np.float32)
idx = g.build_index(D(tgt_s), 0.6)
for it in (1, 2, 5, 64):
    T, info = g.align(D(src), D(cs), idx, D(ct), T0s, max_iter=it, lm=False)
    r = oracle.align(src, cs, tgt_s, ct, T0s, max_iter=it, lm=False)
    print("shifted C1 GN it", it, "gpu dT", T[:3, 3] - T0s[:3, 3], "ref dT", r["T"][:3, 3] - T0s[:3, 3])
sc, mp, src, sub, inb, inb2, T_true, T0 = _c3_cropped(3000)
crop, crop2 = np.ascontiguousarray(mp[inb]), np.ascontiguousarray(mp[inb2])
nb_c, _ = oracle.knn(crop2, crop, 20)
ct_crop = oracle.covariance(crop2, nb_c)[0].astype(np.float32)
nb_s, _ = oracle.knn(sc, src, 20)
cs = oracle.covariance(sc, nb_s)[0].astype(np.float32)
ct_full = np.tile(np.array([1, 0, 0, 1, 0, 1], np.float32), (len(mp), 1))
ct_full[inb] = ct_crop
imap = g.build_index(D(mp), 0.5)
ctd = D(ct_full)
out, _ = g.linearize(D(src), D(cs), imap, ctd, T0, 1.0, pivot=T0[:3, 3])
print("public lin29", out.cpu().numpy())
o29, _, _ = oracle.linearize(src, cs, crop, ct_crop, T0, 1.0, pivot=T0[:3, 3])
print("oracle lin29", o29)
sys.stdout.flush()
os.environ["GICP_DEBUG_ALIGN"] = "1"
T, info = g.align(D(src), D(cs), imap, ctd, T0, max_iter=1, lm=False)
