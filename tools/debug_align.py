"""GPU vs oracle align on C2 with diagnostics."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import gen
import oracle
import paper_2308_07173_b200 as g

D = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731


def perr(T, R):
    dt = np.linalg.norm(T[:3, 3] - R[:3, 3])
    c = (np.trace(T[:3, :3] @ R[:3, :3].T) - 1) / 2
    return dt, math.acos(max(-1, min(1, c)))


src, tgt, T_rel, T0 = gen.config_c2(30000)
ns, _ = oracle.knn(src, src, 20)
nt, _ = oracle.knn(tgt, tgt, 20)
cs = oracle.covariance(src, ns)[0].astype(np.float32)
ct = oracle.covariance(tgt, nt)[0].astype(np.float32)
idx = g.build_index(D(tgt), 0.0)
for lm in (True, False):
    T, info = g.align(D(src), D(cs), idx, D(ct), T0, lm=lm)
    ref = oracle.align(src, cs, tgt, ct, T0, lm=lm)
    eg = oracle.linearize(src, cs, tgt, ct, T, 1.0)[0]
    er = oracle.linearize(src, cs, tgt, ct, ref["T"], 1.0)[0]
    print(f"lm={lm} gpu it={info.iterations} conv={info.converged} err={info.error:.4f} inl={info.inliers}")
    print(f"      ref it={ref['iterations']} conv={ref['converged']} err={ref['error']:.4f} inl={ref['inliers']}")
    print("      pose diff", perr(T, ref["T"]), "vs truth gpu", perr(T, T_rel), "ref", perr(ref["T"], T_rel))
    print(f"      oracle cost at gpu T {eg[27]:.4f} n={eg[28]}  at ref T {er[27]:.4f} n={er[28]}")
# iterate step by step: compare linearize at the same T along the oracle path
T = T0.copy()
for it in range(5):
    o29, ab, corr = oracle.linearize(src, cs, tgt, ct, T, 1.0)
    out, gc = g.linearize(D(src), D(cs), idx, D(ct), T, 1.0)
    h = out.cpu().numpy()
    print(it, "corr equal", np.array_equal(gc.cpu().numpy(), corr), "e", h[27], o29[27], "n", h[28], o29[28],
          "maxrel H", np.abs(h[:21] - o29[:21]).max() / np.abs(o29[:21]).max())
    e2, _ = g.linearize(D(src), D(cs), idx, D(ct), T, 1.0, corr=gc, reuse_corr=True, error_only=True)
    o2 = oracle.linearize(src, cs, tgt, ct, T, 1.0, corr=corr)[0]
    print("   error-only e", e2.cpu().numpy()[27], o2[27])
    # GN step
    H = np.zeros((6, 6)); k = 0
    for a in range(6):
        for b in range(a, 6):
            H[a, b] = H[b, a] = o29[k]; k += 1
    d = np.linalg.solve(H, -o29[21:27])
    T = oracle.se3_exp(d) @ T
