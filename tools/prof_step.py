"""One warm C3 step under cudaProfilerStart/Stop (for ncu --profile-from-start off).
Same launch configuration as bench.py's step."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import gen  # noqa: E402
import paper_2308_07173_b200 as g  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    sc, mp, T_true, T0 = gen.config_c3()
    map_d = torch.from_numpy(np.array(mp)).to(dev)
    scan_d = torch.from_numpy(np.array(sc)).to(dev)
    only = os.environ.get("PROF_ONLY", "")

    def step():
        imap = g.build_index(map_d, bench.MAP_CELL)
        _, _, cov_map = g.knn_cov_self(imap, bench.K, bench.EPS, with_nbr=True)
        g.attach_cov(imap, cov_map)
        iscan = g.build_index(scan_d, 0.0)
        _, _, cov_scan = g.knn_cov_self(iscan, bench.K, bench.EPS, with_nbr=True)
        if only != "knn":
            T, info = g.align(scan_d, cov_scan, imap, cov_map, T0)
        torch.cuda.synchronize()
        imap.free()
        iscan.free()

    for _ in range(2):
        step()
    torch.cuda.cudart().cudaProfilerStart()
    step()
    torch.cuda.cudart().cudaProfilerStop()
    print("prof_step ok")


if __name__ == "__main__":
    main()
