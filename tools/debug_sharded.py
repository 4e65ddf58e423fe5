"""Single-process checks of gicp_align_batched_sharded's allreduce callback path."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from tests.test_gpu_sharded import TINY, SCANS, _problem
from paper_2308_07173_b200 import sharding

for name, scans in (("tiny", TINY), ("scans", SCANS)):
    g, im, cm, src, cov, offs, T0 = _problem(scans)
    plan = sharding.ShardPlan(offs, src.device)
    src_l, cov_l = src.index_select(0, plan.idx), cov.index_select(0, plan.idx)
    res = {}
    for mode in ("none", "roundtrip", "zeros_sync"):
        if mode == "none":
            ar = None
        elif mode == "roundtrip":
            def ar(t):
                h = t.cpu()
                t.copy_(h)
        else:
            def ar(t):
                torch.cuda.synchronize()
                t.add_(torch.zeros_like(t))
        try:
            T, inf = g.align_batched_sharded(src_l, cov_l, plan.loffs, plan.gid, plan.num_chunks, plan.B, im, cm, T0,
                                             allreduce=ar)
            res[mode] = T
            print(name, mode, [(i.iterations, i.inliers) for i in inf])
        except Exception as e:
            print(name, mode, "ERROR", e)
    Tu, iu = g.align_batched(src, cov, offs, im, cm, T0)
    print(name, "unsharded", [(i.iterations, i.inliers) for i in iu])
    if "none" in res and "roundtrip" in res:
        print(name, "none == roundtrip", np.array_equal(res["none"], res["roundtrip"]))
