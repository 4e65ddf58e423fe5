"""Per-kernel device durations of one warm C3 step under torch.profiler (CUPTI
activity records: real cache state, no replay), summed by kernel name.
usage: python tools/kprof.py [steps]"""
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import gen  # noqa: E402
import paper_2308_07173_b200 as g  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
dev = torch.device("cuda", 0)
sc, mp, T_true, T0 = gen.config_c3()
map_d = torch.from_numpy(np.array(mp)).to(dev)
scan_d = torch.from_numpy(np.array(sc)).to(dev)


def step():
    imap = g.build_index(map_d, bench.MAP_CELL)
    _, _, cov_map = g.knn_cov_self(imap, bench.K, bench.EPS, with_nbr=True)
    g.attach_cov(imap, cov_map)
    iscan = g.build_index(scan_d, 0.0)
    _, _, cov_scan = g.knn_cov_self(iscan, bench.K, bench.EPS, with_nbr=True)
    T, info = g.align(scan_d, cov_scan, imap, cov_map, T0)
    imap.free()
    iscan.free()
    return info


for _ in range(3):
    step()
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for _ in range(steps):
        info = step()
    torch.cuda.synchronize()
agg = defaultdict(lambda: [0, 0.0])
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        agg[e.name[:70]][0] += 1
        agg[e.name[:70]][1] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
tot = sum(v[1] for v in agg.values())
print(f"align iterations {info.iterations}; device total {tot / steps:.1f} us/step")
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"{t / steps:9.1f} us {100 * t / tot:5.1f}% n={n // steps:4d} avg {t / n:7.1f}  {k}")
