"""The C4 batch aligned as one batched call vs G concurrent calls (host threads, own
streams) over disjoint groups of registrations: time and bitwise pose check.
usage: python tools/c4_halves.py [n_distinct] [G,...]"""
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
import gen
import paper_2308_07173_b200 as g
from paper_2308_07173_b200 import sharding

nd = int(sys.argv[1]) if len(sys.argv) > 1 else 32
Gs = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1,2,4").split(",")]
scans = bench.gen_scans(list(range(nd)), min(nd, os.cpu_count() or 1))
mp = gen.racetrack_map(2_000_000, 1)
dev = torch.device("cuda:0")
md = torch.from_numpy(mp).to(dev)
sd = torch.from_numpy(np.concatenate([s for s, _ in scans])).to(dev)
imap = g.build_index(md, bench.MAP_CELL)
_, _, cm = g.knn_cov_self(imap, 20, 1e-3)
g.attach_cov(imap, cm)
cs = torch.empty((nd * bench.N_SCAN, 6), dtype=torch.float32, device=dev)
for i in range(nd):
    isc = g.build_index(sd[i * bench.N_SCAN:(i + 1) * bench.N_SCAN], 0.0)
    g.knn_cov_self(isc, 20, 1e-3, out=(None, None, cs[i * bench.N_SCAN:(i + 1) * bench.N_SCAN]))
B = nd * bench.N_HYP
_, T0 = bench.c4_poses()
T0 = np.asarray(T0[:B])
ref = None
for G in Gs:
    per = B // G
    groups = [list(range(k * per, (k + 1) * per)) for k in range(G)]
    streams = [torch.cuda.Stream(device=dev) for _ in range(G)]
    plans = []
    for k, regs in enumerate(groups):
        offs = np.arange(len(regs) + 1, dtype=np.int64) * bench.N_SCAN
        rb = (np.asarray(regs) // bench.N_HYP) * bench.N_SCAN
        plans.append((offs, sharding.ShardPlan(offs, dev, reg_base=rb)))
    pool = ThreadPoolExecutor(max_workers=G, initializer=lambda: torch.cuda.set_device(0))

    def job(k):
        with torch.cuda.stream(streams[k]):
            offs, plan = plans[k]
            T, infos = sharding.align_batched_sharded(g, sd, cs, offs, imap, cm, T0[groups[k]], plan=plan)
            streams[k].synchronize()
            return np.asarray(T)
    best = 1e9
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        Ts = list(pool.map(job, range(G)))
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    T = np.concatenate(Ts)
    same = ref is None or np.array_equal(T, ref)
    ref = T if ref is None else ref
    print(f"RESULT G={G}: align {best * 1e3:.2f} ms, poses bitwise equal to G={Gs[0]}: {same}", flush=True)
