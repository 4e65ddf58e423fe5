"""L2 bandwidth (SURVEY §5/§8(d) asks for it; the kNN's candidate re-reads are L2 hits):
torch reductions and copies over buffers that fit the 126 MB L2 (repeated, so every
pass after the first hits L2) vs the same over 2 GB (HBM). CUDA events; prints JSON."""
import json

import torch

dev = torch.device("cuda:0")
props = torch.cuda.get_device_properties(dev)
res = {"device": props.name, "l2_bytes": getattr(props, "L2_cache_size", None), "sm_count": props.multi_processor_count}


def timeit(fn, reps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e-3


for mb in (16, 32, 48, 1024):
    n = mb * (1 << 20) // 4
    x = torch.rand(n, device=dev)
    y = torch.empty_like(x)
    t_sum = timeit(lambda: x.sum())
    t_cp = timeit(lambda: y.copy_(x))
    res[f"read_{mb}MB_GBps"] = x.numel() * 4 / t_sum / 1e9
    res[f"copy_{mb}MB_GBps (read+write)"] = 2 * x.numel() * 4 / t_cp / 1e9
print(json.dumps(res))
