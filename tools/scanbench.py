"""Time the C3 scan path (auto-cell index build + kNN+cov, k=20) and report the
escalation count. usage: GICP_LIB_VARIANT=... python tools/scanbench.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import gen
import paper_2308_07173_b200 as g

sc, mp, T, T0 = gen.config_c3()
sd = torch.from_numpy(np.array(sc)).cuda()
for name, src in (("C3 scan", sd), ("C2 scan", torch.from_numpy(np.array(gen.config_c2()[0])).cuda())):
    tb, tk = [], []
    for r in range(12):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record()
        isc = g.build_index(src, 0.0)
        e[1].record()
        g.knn_cov_self(isc, 20, 1e-3)
        e[2].record()
        torch.cuda.synchronize()
        if r >= 2:
            tb.append(e[0].elapsed_time(e[1]))
            tk.append(e[1].elapsed_time(e[2]))
        info = isc
        isc.free()
    print(f"{os.path.basename(os.environ.get('GICP_LIB_VARIANT', 'default'))} {name}: cell {info.cell_size:.3f} "
          f"voxels {info.n_cells} build {np.median(tb):.3f} ms knn_cov {np.median(tk):.3f} ms")
