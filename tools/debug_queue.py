import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen, oracle, paper_2308_07173_b200 as g
D = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
src, tgt, T_true, T0 = gen.config_c1(sigma=0.002)
cs = oracle.covariance(src, oracle.knn(src, src, 10)[0])[0].astype(np.float32)
ct = oracle.covariance(tgt, oracle.knn(tgt, tgt, 10)[0])[0].astype(np.float32)
idx = g.build_index(D(tgt), 0.6)
for nc in ("0", "1"):
    os.environ["GICP_ALIGN_NOCACHE"] = nc
    T, info = g.align(D(src), D(cs), idx, D(ct), T0)
    torch.cuda.synchronize()
    print("nocache", nc, info, T[:3, 3], flush=True)
r = oracle.align(src, cs, tgt, ct, T0)
print("oracle", r["iterations"], r["T"][:3, 3])
