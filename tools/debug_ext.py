"""EXT tile kNN vs the per-query path (GICP_KNN_TILE=0) on external queries."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import os, sys, numpy as np, torch
sys.path.insert(0, os.environ["ROOT"])
import gen, paper_2308_07173_b200 as g
which = os.environ["WHICH"]
if which == "c5":
    mp, q = gen.config_c5(); cell = 0.2; k = 32
else:
    mp = gen.racetrack_map(300_000, 3); sc, T = gen.scan(20_000, 700.0, 2001)
    q = gen.apply_T(T, sc).astype(np.float32); cell = 0.4; k = 20
idx = g.build_index(torch.from_numpy(np.ascontiguousarray(mp)).cuda(), cell)
os.environ["GICP_DEBUG_STATS"] = "1"
n, d = g.knn(idx, torch.from_numpy(q).cuda(), k)
np.save("/tmp/ext_%s_%s_n.npy" % (which, os.environ.get("GICP_KNN_TILE", "1")), n.cpu().numpy())
np.save("/tmp/ext_%s_%s_d.npy" % (which, os.environ.get("GICP_KNN_TILE", "1")), d.cpu().numpy())
np.save("/tmp/ext_%s_q.npy" % which, q)
'''
for which in ("c5",):
    for tile in ("0", "1"):
        r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, ROOT=ROOT, WHICH=which, GICP_KNN_TILE=tile),
                           capture_output=True, text=True)
        print(which, tile, [l for l in r.stderr.splitlines() if "gicp knn" in l or "Error" in l][:3])
    import numpy as np
    a_n, a_d = np.load(f"/tmp/ext_{which}_0_n.npy"), np.load(f"/tmp/ext_{which}_0_d.npy")
    b_n, b_d = np.load(f"/tmp/ext_{which}_1_n.npy"), np.load(f"/tmp/ext_{which}_1_d.npy")
    bad = np.nonzero(np.any(a_n != b_n, axis=1) | np.any(a_d.view(np.uint32) != b_d.view(np.uint32), axis=1))[0]
    print(which, "rows differing", len(bad), "of", len(a_n))
    for r in bad[:3]:
        print("  row", r, "ref d2", a_d[r][:8], "\n        got d2", b_d[r][:8], "\n  ref n", a_n[r][:8], "\n  got n", b_n[r][:8])
