"""C3 cropped fixture: the first align iterations, GPU vs oracle (GN and LM)."""
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
np.set_printoptions(precision=6, suppress=True)
for lm in (False, True):
    for it in (1, 2, 3):
        T, info = g.align(D(src), D(cs), imap, ctd, T0, max_iter=it, lm=lm)
        r = oracle.align(src, cs, crop, ct_crop, T0, max_iter=it, lm=lm)
        print(f"lm={lm} it={it} gpu dT {T[:3, 3] - T0[:3, 3]} err {info.error:.4f} | ref dT {r['T'][:3, 3] - T0[:3, 3]} err {r['error']:.4f}")
# the same with the source in a different order (the align sorts a copy)
perm = np.random.default_rng(1).permutation(len(src))
T, info = g.align(D(src[perm]), D(cs[perm]), imap, ctd, T0, max_iter=1, lm=False)
print("permuted source GN it=1 dT", T[:3, 3] - T0[:3, 3])
# python GN step from the public linearize
out, _ = g.linearize(D(src), D(cs), imap, ctd, T0, 1.0, pivot=T0[:3, 3])
h = out.cpu().numpy()
H = np.zeros((6, 6)); k = 0
for a in range(6):
    for c in range(a, 6):
        H[a, c] = H[c, a] = h[k]; k += 1
d = np.linalg.solve(H, -h[21:27])
print("public-linearize GN delta", d)
