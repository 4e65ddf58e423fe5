import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen, paper_2308_07173_b200 as g
D = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
mp = gen.racetrack_map(2_000_000, 1)
im = g.build_index(D(mp), 0.5)
_, _, cm = g.knn_cov_self(im, 20, 1e-3)
g.attach_cov(im, cm)
sc, T, Tp = gen.config_c4_scan(0, 20000)
sd = D(sc)
isc = g.build_index(sd, 0.0)
_, _, cs = g.knn_cov_self(isc, 20, 1e-3)
os.environ["GICP_DEBUG_ALIGN"] = "1"
for nc in ("1", "0"):
    os.environ["GICP_ALIGN_NOCACHE"] = nc
    print("=== nocache", nc, "single", flush=True)
    T1, i1 = g.align(sd, cs, im, cm, Tp, max_iter=6)
    torch.cuda.synchronize(); sys.stderr.flush()
    print("=== nocache", nc, "batched", flush=True)
    Tb, ib = g.align_batched(sd, cs, [0, len(sc)], im, cm, Tp[None], max_iter=6)
    torch.cuda.synchronize(); sys.stderr.flush()
    print("equal", np.array_equal(Tb[0], T1), i1, ib[0], flush=True)
