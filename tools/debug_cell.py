"""Exactness across index cells: the 1-NN is exact, so corr/out29 of a
linearisation and the poses of an align must be bitwise the same for any map
cell. Finds the first difference."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
import gen
import paper_2308_07173_b200 as g
from paper_2308_07173_b200 import sharding

cells = [float(c) for c in (sys.argv[1] if len(sys.argv) > 1 else "0.5,0.4").split(",")]
dev = torch.device("cuda:0")
scans = bench.gen_scans([0], 1)
mp = gen.racetrack_map(2_000_000, 1)
md = torch.from_numpy(mp).to(dev)
sd = torch.from_numpy(scans[0][0]).to(dev)
imap = g.build_index(md, bench.MAP_CELL)
_, _, cm = g.knn_cov_self(imap, 20, 1e-3)
isc = g.build_index(sd, 0.0)
_, _, cs = g.knn_cov_self(isc, 20, 1e-3)
_, T0 = bench.c4_poses()
idx = {}
for c in cells:
    idx[c] = g.build_index(md, c)
    g.attach_cov(idx[c], cm)
H = lambda t: t.cpu().numpy()
# (1) single linearisations at the 8 initial poses and along the first align
ref = cells[0]
for h in range(8):
    outs = {c: g.linearize(sd, cs, idx[c], cm, T0[h], 1.0) for c in cells}
    for c in cells[1:]:
        dc = np.flatnonzero(H(outs[c][1]) != H(outs[ref][1]))
        do = np.abs(H(outs[c][0]) - H(outs[ref][0])).max()
        print(f"lin T0[{h}] cell {c}: corr diffs {len(dc)} out29 maxdiff {do:.3e}", dc[:5])
        if len(dc):
            i = dc[0]
            print("   point", i, "corr", H(outs[ref][1])[i], H(outs[c][1])[i])
# (2) single aligns
for h in range(8):
    res = {c: g.align(sd, cs, idx[c], cm, T0[h]) for c in cells}
    for c in cells[1:]:
        d = np.abs(res[c][0] - res[ref][0]).max()
        print(f"align T0[{h}] cell {c}: |dT| {d:.3e} iters {res[ref][1].iterations} {res[c][1].iterations}")
# (3) batched 8
offsets = np.arange(9, dtype=np.int64) * bench.N_SCAN
sd8 = sd.repeat(1, 1)
plan = sharding.ShardPlan(offsets, dev, reg_base=np.zeros(8, np.int64))
resb = {c: sharding.align_batched_sharded(g, sd, cs, offsets, idx[c], cm, T0[:8], plan=plan) for c in cells}
for c in cells[1:]:
    Tb = np.asarray(resb[c][0]); Tr = np.asarray(resb[ref][0])
    print(f"batched cell {c}: per-reg |dT|", [f"{np.abs(Tb[b] - Tr[b]).max():.1e}" for b in range(8)])
