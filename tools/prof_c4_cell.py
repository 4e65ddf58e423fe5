"""The reduced C4 batch (tools/prof_c4.py) aligned against map indexes built with
different level-0 cells (the 1-NN search is exact, so the poses must be bitwise
the same for every cell): align time and per-kind linearisation launch times.
usage: python tools/prof_c4_cell.py n_distinct cell[,cell...]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
import gen
import paper_2308_07173_b200 as g
from paper_2308_07173_b200 import sharding

nd = int(sys.argv[1]) if len(sys.argv) > 1 else 8
cells = [float(c) for c in (sys.argv[2] if len(sys.argv) > 2 else "0.5").split(",")]
scans = bench.gen_scans(list(range(nd)), min(nd, os.cpu_count() or 1))
mp = gen.racetrack_map(2_000_000, 1)
dev = torch.device("cuda:0")
md = torch.from_numpy(mp).to(dev)
sd = torch.from_numpy(np.concatenate([s for s, _ in scans])).to(dev)
imap = g.build_index(md, bench.MAP_CELL)
_, _, cm = g.knn_cov_self(imap, 20, 1e-3)
cs = torch.empty((nd * bench.N_SCAN, 6), dtype=torch.float32, device=dev)
for i in range(nd):
    isc = g.build_index(sd[i * bench.N_SCAN:(i + 1) * bench.N_SCAN], 0.0)
    g.knn_cov_self(isc, 20, 1e-3, out=(None, None, cs[i * bench.N_SCAN:(i + 1) * bench.N_SCAN]))
B = nd * bench.N_HYP
_, T0 = bench.c4_poses()
T0 = T0[:B]
offsets = np.arange(B + 1, dtype=np.int64) * bench.N_SCAN
plan = sharding.ShardPlan(offsets, dev, reg_base=(np.arange(B) // bench.N_HYP) * bench.N_SCAN)
ref = None
for cell in cells:
    it = g.build_index(md, cell)
    g.attach_cov(it, cm)
    sharding.align_batched_sharded(g, sd, cs, offsets, it, cm, T0, plan=plan)  # warm-up
    torch.cuda.synchronize()
    best = 1e9
    for rep in range(3):
        g.align_timing(rep == 2)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        T, infos = sharding.align_batched_sharded(g, sd, cs, offsets, it, cm, T0, plan=plan)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    ms, n, pts = g.align_timing(False)
    T = np.asarray(T)
    same = ref is None or np.array_equal(T, ref)
    ref = T if ref is None else ref
    print(f"RESULT cell={cell} align {best * 1e3:.2f} ms iters {sum(i.iterations for i in infos)} "
          f"bitwise_same_as_first={same}")
    for k in range(3):
        if n[k]:
            print(f"  kind {k}: {ms[k] / n[k]:.3f} ms/launch, {pts[k] / n[k]:.0f} pts/launch, "
                  f"{80 * pts[k] / (ms[k] * 1e-3) / 1e9:.1f} GB/s, total {ms[k]:.2f} ms")
    sys.stdout.flush()
