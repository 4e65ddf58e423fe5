"""GPU vs oracle on the C3 cropped-align fixture (tests/test_gpu_pins.py): linearize at
T0 and along the oracle's path, then both aligns with the GPU's per-iteration trace."""
import math
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
n_sub = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
sc, mp, src, sub, inb, inb2, T_true, T0 = _c3_cropped(n_sub)
crop, crop2 = np.ascontiguousarray(mp[inb]), np.ascontiguousarray(mp[inb2])
nb_c, _ = oracle.knn(crop2, crop, 20)
ct_crop = oracle.covariance(crop2, nb_c)[0].astype(np.float32)
nb_s, _ = oracle.knn(sc, src, 20)
cs = oracle.covariance(sc, nb_s)[0].astype(np.float32)
ct_full = np.tile(np.array([1, 0, 0, 1, 0, 1], np.float32), (len(mp), 1))
ct_full[inb] = ct_crop
crop_ids = np.nonzero(inb)[0]
imap = g.build_index(D(mp), 0.5)
ctd = D(ct_full)
for attach in (False, True):
    if attach:
        g.attach_cov(imap, ctd)
    for T in (T0, T_true):
        piv = T[:3, 3]
        out, gc = g.linearize(D(src), D(cs), imap, ctd, T, 1.0, pivot=piv)
        o29, ab, corr = oracle.linearize(src, cs, crop, ct_crop, T, 1.0, pivot=piv)
        h = out.cpu().numpy()
        gcn = gc.cpu().numpy()
        ref_corr = np.where(corr >= 0, crop_ids[np.maximum(corr, 0)], -1)
        print(f"attach={attach} corr equal {np.array_equal(gcn, ref_corr)} (mismatch {(gcn != ref_corr).sum()}) "
              f"n {h[28]} {o29[28]} e {h[27]:.6f} {o29[27]:.6f} maxrel H "
              f"{np.abs(h[:21] - o29[:21]).max() / np.abs(o29[:21]).max():.3g} b {h[21:27]} {o29[21:27]}")
for nocache in ("0", "1"):
    os.environ["GICP_ALIGN_NOCACHE"] = nocache
    os.environ["GICP_DEBUG_ALIGN"] = "1"
    T, info = g.align(D(src), D(cs), imap, ctd, T0)
    sys.stderr.flush()
    print("nocache", nocache, "gpu it", info.iterations, "dt_true", np.linalg.norm(T[:3, 3] - T_true[:3, 3]))
os.environ.pop("GICP_DEBUG_ALIGN")
r = oracle.align(src, cs, crop, ct_crop, T0, trace=True)
print("oracle it", r["iterations"], "dt_true", np.linalg.norm(r["T"][:3, 3] - T_true[:3, 3]))
for row in r["trace"]:
    print("  it %d lam %.3e e %.6f en %.6f rho %.3g" % (row[0], row[1], row[2], row[3], row[4]))
