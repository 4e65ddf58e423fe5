"""Time the C3 map / scan self kNN(k=20)+cov for several cell sizes and library
variants (GICP_LIB_VARIANT), one subprocess each.
usage: python tools/knn_sweep.py cells=0.45,0.5 libs=default,variants/libgicp_x.so envs=A=1,A=0 (';'-separated sets)"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
args = dict(a.split("=", 1) for a in sys.argv[1:])
cells = args.get("cells", "0.5").split(",")
libs = args.get("libs", "default").split(",")
code = r'''
import os, sys, numpy as np, torch
sys.path.insert(0, os.environ["ROOT"])
import gen, paper_2308_07173_b200 as g
cell = float(os.environ["CELL"])
sc, mp, T, T0 = gen.config_c3()
for name, pts, c in (("map", mp, cell), ("scan", sc, float(os.environ.get("SCAN_CELL", "0")))):
    if name == "scan" and os.environ.get("SCAN", "1") == "0": continue
    idx = g.build_index(torch.from_numpy(np.array(pts)).cuda(), c)
    n = len(pts)
    out = (torch.empty((n, 20), dtype=torch.int32, device="cuda"), torch.empty((n, 20), dtype=torch.float32, device="cuda"),
           torch.empty((n, 6), dtype=torch.float32, device="cuda"))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ts = []
    for r in range(13):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); g.knn_cov_self(idx, 20, 1e-3, out=out); b.record(); torch.cuda.synchronize()
        if r >= 3: ts.append(a.elapsed_time(b))
    os.environ["GICP_DEBUG_STATS"] = "1"
    g.knn_cov_self(idx, 20, 1e-3, out=out); torch.cuda.synchronize()
    os.environ.pop("GICP_DEBUG_STATS")
    print(f"RESULT {os.path.basename(os.environ.get('GICP_LIB_VARIANT', 'default'))} {name} cell={idx.cell_size:.3f} median {np.median(ts):.3f} ms min {np.min(ts):.3f}", flush=True)
'''
envs = [e for e in args.get("envs", "").split(";")]
for lib in libs:
  for es in envs:
    extra = dict(kv.split("=", 1) for kv in es.split(",") if kv)
    for cell in cells:
        env = dict(os.environ, ROOT=ROOT, CELL=cell, **extra)
        print("ENV", es, flush=True)
        if lib != "default":
            env["GICP_LIB_VARIANT"] = os.path.join(ROOT, "paper_2308_07173_b200", lib)
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
        for ln in (r.stdout + r.stderr).splitlines():
            if ln.startswith("RESULT") or ln.startswith("[gicp knn]") or "Error" in ln:
                print(ln, flush=True)
