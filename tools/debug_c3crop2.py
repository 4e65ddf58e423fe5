"""C3 cropped fixture: GPU align under cube-stage variants vs the oracle."""
import os
import subprocess
import sys

code = r'''
import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import gen, oracle, paper_2308_07173_b200 as g
from tests.test_gpu_pins import _c3_cropped
D = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
sc, mp, src, sub, inb, inb2, T_true, T0 = _c3_cropped(3000)
crop, crop2 = np.ascontiguousarray(mp[inb]), np.ascontiguousarray(mp[inb2])
nb_c, _ = oracle.knn(crop2, crop, 20)
ct_crop = oracle.covariance(crop2, nb_c)[0].astype(np.float32)
nb_s, _ = oracle.knn(sc, src, 20)
cs = oracle.covariance(sc, nb_s)[0].astype(np.float32)
ct_full = np.tile(np.array([1, 0, 0, 1, 0, 1], np.float32), (len(mp), 1))
ct_full[inb] = ct_crop
imap = g.build_index(D(mp), 0.5)
ctd = D(ct_full)
if os.environ.get("ATTACH") == "1":
    g.attach_cov(imap, ctd)
T, info = g.align(D(src), D(cs), imap, ctd, T0)
print(os.environ.get("GICP_LIN_COARSE_THR"), os.environ.get("ATTACH"), "gpu it", info.iterations, "dt_true", np.linalg.norm(T[:3, 3] - T_true[:3, 3]))
'''
for thr in ("1e9", "0.4", "0"):
    for att in ("0", "1"):
        env = dict(os.environ, GICP_LIN_COARSE_THR=thr, ATTACH=att)
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
        print(r.stdout.strip(), r.stderr.strip()[-300:] if r.returncode else "")
        sys.stdout.flush()
