"""Why do some C4 registrations run to max_iter? GICP_DEBUG_ALIGN trace of one."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from tests.test_gpu_sharded import SCANS, _problem

g, im, cm, src, cov, offs, T0 = _problem(SCANS)
os.environ["GICP_DEBUG_ALIGN"] = "1"
for b in (0, 2):
    s, c = src[offs[b]:offs[b + 1]].contiguous(), cov[offs[b]:offs[b + 1]].contiguous()
    T, info = g.align(s, c, im, cm, T0[b])
    torch.cuda.synchronize()
    sys.stderr.flush()
    print("reg", b, info, flush=True)
