"""Time gicp_linearize on C3 (100k scan vs 2M map) at T_true and at T0."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import gen
import paper_2308_07173_b200 as g

sc, mp, T, T0 = gen.config_c3()
md = torch.from_numpy(np.array(mp)).cuda()
if os.environ.get("LB_SORT"):  # Morton-sort the source as gicp_align does
    c = np.floor(sc / 0.5).astype(np.int64) + (1 << 20)
    def spread(v):
        v = v & 0x1fffff
        r = np.zeros_like(v)
        for b in range(21):
            r |= ((v >> b) & 1) << (3 * b)
        return r
    key = spread(c[:, 0]) | (spread(c[:, 1]) << 1) | (spread(c[:, 2]) << 2)
    sc = np.ascontiguousarray(sc[np.argsort(key, kind="stable")])
sd = torch.from_numpy(np.array(sc)).cuda()
im = g.build_index(md, 0.5)
cm = torch.from_numpy(gen.random_covariances(len(mp), 2)).cuda()
cs = torch.from_numpy(gen.random_covariances(len(sc), 1)).cuda()
if os.environ.get("LB_REALCOV"):
    _, _, cm = g.knn_cov_self(im, 20, 1e-3)
    isc = g.build_index(sd, 0.0)
    _, _, cs = g.knn_cov_self(isc, 20, 1e-3)
if os.environ.get("LB_ALIGN"):
    for it in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        Tr, info = g.align(sd, cs, im, cm, T0)
        b.record()
        torch.cuda.synchronize()
        print(f"align: {a.elapsed_time(b):.2f} ms, {info.iterations} it, converged {info.converged}, "
              f"|dt| {np.linalg.norm(Tr[:3, 3] - T[:3, 3]):.4f}")
out = torch.empty(29, dtype=torch.float64, device="cuda")
if os.environ.get("LB_ATTACH"):
    g.attach_cov(im, cm)
corr = torch.empty(len(sc), dtype=torch.int32, device="cuda")
prof = os.environ.get("LB_PROF")
for name, TT, kw in (("T_true", T, {}), ("T0", T0, {}), ("T_true reuse+err", T, dict(reuse_corr=True, error_only=True))):
    ts = []
    for r in range(12):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if prof and r == 11:
            torch.cuda.cudart().cudaProfilerStart()
        a.record()
        g.linearize(sd, cs, im, cm, TT, 1.0, corr=corr, out=out, **kw)
        b.record()
        torch.cuda.synchronize()
        if prof and r == 11:
            torch.cuda.cudart().cudaProfilerStop()
        if r >= 2:
            ts.append(a.elapsed_time(b))
    print(f"linearize {name}: median {1e3 * np.median(ts):.1f} us  inliers {out[28].item():.0f}")
# back-to-back launches: per-call device time once the queue is ahead of the GPU
for name, TT, kw in (("T_true", T, {}), ("T0", T0, {}), ("T_true reuse+err", T, dict(reuse_corr=True, error_only=True))):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g.linearize(sd, cs, im, cm, TT, 1.0, corr=corr, out=out, **kw)
    torch.cuda._sleep(2_000_000)
    a.record()
    for r in range(50):
        g.linearize(sd, cs, im, cm, TT, 1.0, corr=corr, out=out, **kw)
    b.record()
    torch.cuda.synchronize()
    print(f"linearize {name} x50 loop: {1e3 * a.elapsed_time(b) / 50:.1f} us/call")
