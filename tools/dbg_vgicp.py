import sys; sys.path.insert(0, '.')
import numpy as np, torch, gen, oracle as orc
import paper_2308_07173_b200 as g
D = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
src, tgt, T_true, T0 = gen.config_c1(sigma=0.0)
ns, _ = orc.knn(src, src, 10); nt, _ = orc.knn(tgt, tgt, 10)
cs = orc.covariance(src, ns)[0].astype(np.float32); ct = orc.covariance(tgt, nt)[0].astype(np.float32)
idx = g.build_index(D(tgt), 0.5); g.attach_voxels(idx, D(ct))
T = T0.copy()
for it in range(8):
    piv = T[:3, 3]
    o = g.linearize_vgicp(D(src), D(cs), idx, T, 7, pivot=piv).cpu().numpy()
    r, ab = orc.linearize_vgicp(src, cs, tgt, ct, T, 0.5, 7, pivot=piv)
    print(it, o[27], r[27], o[28], r[28], np.abs(o[:27]-r[:27]).max())
    # GN step from oracle
    H = np.zeros((6,6)); k=0
    for a in range(6):
        for c in range(a,6): H[a,c]=H[c,a]=r[k]; k+=1
    d = np.linalg.solve(H, -r[21:27])
    T = orc.pivoted_exp(d, piv) @ T
Tg, info = g.align_vgicp(D(src), D(cs), idx, T0, 7)
print(info, Tg[:3,3])
rr = orc.align_vgicp(src, cs, tgt, ct, T0, 0.5, 7); print(rr['iterations'], rr['converged'], rr['T'][:3,3])
