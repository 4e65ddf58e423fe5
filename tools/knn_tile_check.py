"""A/B of the tiled self-kNN stage (GICP_KNN_TILE=0 disables it): C3 map and scan
outputs compared across the two paths (nbr, d2 bitwise; covariances), times.
usage: python tools/knn_tile_check.py [cell]"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import os, sys, numpy as np, torch
sys.path.insert(0, os.environ["ROOT"])
import gen, paper_2308_07173_b200 as g
cell = float(os.environ.get("CELL", "0.5"))
sc, mp, T, T0 = gen.config_c3()
res = {}
for name, pts, c in (("map", mp, cell), ("scan", sc, 0.0)):
    idx = g.build_index(torch.from_numpy(np.array(pts)).cuda(), c)
    n = len(pts)
    out = (torch.empty((n, 20), dtype=torch.int32, device="cuda"), torch.empty((n, 20), dtype=torch.float32, device="cuda"),
           torch.empty((n, 6), dtype=torch.float32, device="cuda"))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ts = []
    for r in range(12):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); g.knn_cov_self(idx, 20, 1e-3, out=out); b.record(); torch.cuda.synchronize()
        if r >= 2: ts.append(a.elapsed_time(b))
    if os.environ.get("STATS"):
        os.environ["GICP_DEBUG_STATS"] = "1"
        g.knn_cov_self(idx, 20, 1e-3, out=out); torch.cuda.synchronize()
        os.environ.pop("GICP_DEBUG_STATS")
    print(f"{name} tile={os.environ.get('GICP_KNN_TILE', '1')} cell={idx.cell_size:.3f} median {np.median(ts):.3f} ms min {np.min(ts):.3f}", flush=True)
    np.save(f"/tmp/knn_{name}_{os.environ.get('GICP_KNN_TILE', '1')}_nbr.npy", out[0].cpu().numpy())
    np.save(f"/tmp/knn_{name}_{os.environ.get('GICP_KNN_TILE', '1')}_d2.npy", out[1].cpu().numpy())
    np.save(f"/tmp/knn_{name}_{os.environ.get('GICP_KNN_TILE', '1')}_cov.npy", out[2].cpu().numpy())
'''
cell = sys.argv[1] if len(sys.argv) > 1 else "0.5"
for tile in ("0", "1"):
    env = dict(os.environ, ROOT=ROOT, GICP_KNN_TILE=tile, CELL=cell, STATS="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print(r.stdout, r.stderr[-3000:])
import numpy as np
for name in ("map", "scan"):
    a = [np.load(f"/tmp/knn_{name}_0_{x}.npy") for x in ("nbr", "d2", "cov")]
    b = [np.load(f"/tmp/knn_{name}_1_{x}.npy") for x in ("nbr", "d2", "cov")]
    bad = np.nonzero(np.any(a[0] != b[0], axis=1) | np.any(a[1].view(np.uint32) != b[1].view(np.uint32), axis=1))[0]
    print(name, "rows differing (nbr/d2):", len(bad), bad[:10], "max |dcov|", np.abs(a[2] - b[2]).max())
