"""Device-timed numbers for the non-headline configs:
  C2  scan-to-scan latency: index + kNN/cov of both 30k scans + align
  C4  batched registration: B scans x 100k vs the 2M map, gicp_align_batched
      (iterations/s = sum of per-scan iterations / time) vs B single aligns
  C5  20M multi-lap map, 1M queries, k=32: index build, kNN, covariances
usage: python tools/workloads.py [c2] [c4 [B]] [c5]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import gen
import paper_2308_07173_b200 as g

DEV = torch.device("cuda", 0)


def D(a):
    return torch.from_numpy(np.array(a)).to(DEV)


def timed(fn, reps=5, warm=2):
    ts = []
    for r in range(reps + warm):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        out = fn()
        b.record()
        torch.cuda.synchronize()
        if r >= warm:
            ts.append(a.elapsed_time(b))
    return float(np.median(ts)), out


def c2():
    src, tgt, T_rel, T0 = gen.config_c2()
    sd, td = D(src), D(tgt)

    def run():
        it = g.build_index(td, 0.0)
        _, _, ct = g.knn_cov_self(it, 20, with_nbr=False)
        isd = g.build_index(sd, 0.0)
        _, _, cs = g.knn_cov_self(isd, 20, with_nbr=False)
        T, info = g.align(sd, cs, it, ct, T0)
        it.free()
        isd.free()
        return info
    ms, info = timed(run)
    print(json.dumps({"workload": "C2 scan-to-scan 30k vs 30k, k=20", "latency_ms": ms,
                      "align_iterations": info.iterations}))


def c4(B):
    mp = gen.racetrack_map(2_000_000, 1)
    im = g.build_index(D(mp), 0.5)
    _, _, cm = g.knn_cov_self(im, 20, with_nbr=False)
    g.attach_cov(im, cm)
    scans, covs, T0s = [], [], []
    for i in range(B):
        sc, T, T0 = gen.config_c4_scan(i * (256 // B))
        sd = D(sc)
        isc = g.build_index(sd, 0.0)
        _, _, cs = g.knn_cov_self(isc, 20, with_nbr=False)
        isc.free()
        scans.append(sd)
        covs.append(cs)
        T0s.append(T0)
    offs = np.concatenate([[0], np.cumsum([s.shape[0] for s in scans])])
    src = torch.cat(scans).contiguous()
    cov = torch.cat(covs).contiguous()
    T0s = np.array(T0s)
    ms_b, (Ts, infos) = timed(lambda: g.align_batched(src, cov, offs, im, cm, T0s, allow_degenerate=True), reps=3)
    its = sum(i.iterations for i in infos)

    def singles():
        return [g.align(scans[b], covs[b], im, cm, T0s[b])[1] for b in range(B)]
    ms_s, infos_s = timed(singles, reps=3)
    same = all(a.iterations == b.iterations and a.error == b.error for a, b in zip(infos, infos_s))
    print(json.dumps({"workload": f"C4 batched: {B} scans x 100k vs 2M map", "batched_ms": ms_b,
                      "iterations_total": its, "batched_iters_per_s": 1e3 * its / ms_b,
                      "batched_source_pts_per_s": 1e3 * its * 100_000 / ms_b, "singles_ms": ms_s,
                      "singles_iters_per_s": 1e3 * its / ms_s, "identical_to_singles": same}))


def c5():
    t = time.time()
    mp, q = gen.config_c5()
    gen_s = time.time() - t
    mpd, qd = D(mp), D(q)
    ms_build, idx = timed(lambda: g.build_index(mpd, 0.2), reps=3)
    nbr = torch.empty((q.shape[0], 32), dtype=torch.int32, device=DEV)
    d2 = torch.empty((q.shape[0], 32), dtype=torch.float32, device=DEV)
    cov = torch.empty((q.shape[0], 6), dtype=torch.float32, device=DEV)
    ms_knn, _ = timed(lambda: g.knn(idx, qd, 32, out=(nbr, d2)))
    ms_cov, _ = timed(lambda: g.covariances(mpd, nbr, 1e-3, out=cov))
    m = q.shape[0]
    # algorithmic bytes: 12 + 12k + 24 per external query plus 28 B per
    # distinct map point the neighbour sets touch (16 B float4 + 12 B xyz for the covariance)
    uniq = int(torch.unique(nbr).numel())
    alg = m * (12 + 12 * 32 + 24) + 28 * uniq
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(os.path.join(
        os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")) else 6650.0
    ach = alg / ((ms_knn + ms_cov) * 1e-3) / 1e9
    print(json.dumps({"workload": "C5 20M multi-lap map, 1M queries, k=32", "index_build_ms": ms_build,
                      "knn_ms": ms_knn, "cov_ms": ms_cov, "knn_cov_pts_per_s": 1e3 * m / (ms_knn + ms_cov),
                      "algorithmic_bytes": alg, "distinct_map_points": uniq, "achieved_GBps": ach,
                      "roofline_frac": ach / peak, "gen_s": gen_s}))




def kd():
    """kernel-descriptor covariances on the C3 map (2M, k=20), per kernel x reg."""
    mp = gen.racetrack_map(2_000_000, 1)
    md = D(mp)
    im = g.build_index(md, 0.5)
    nbr, _, _ = g.knn_cov_self(im, 20)
    o = tuple(float(v) for v in mp.min(axis=0))
    cov = torch.empty((mp.shape[0], 6), dtype=torch.float32, device=DEV)
    res = {}
    ms0, _ = timed(lambda: g.covariances(md, nbr, 1e-3, out=cov))
    res["unweighted_plane"] = ms0
    for kern, sig in (("laplacian", 0.5), ("rbf", 4.0), ("gaussian", 0.3), ("polynomial", 1.0), ("hi", 1.0)):
        for reg in ("plane", "min_eig"):
            ms, _ = timed(lambda: g.covariances_kd(md, nbr, kern, sigma=sig, alpha=0.01, c=1.0, origin=o, reg=reg,
                                                   out=cov))
            res[f"{kern}_{reg}"] = ms
    print(json.dumps({"workload": "kernel-descriptor covariances, C3 map 2M x k=20 (ms per call)", **res}))


def vg():
    """VGICP on C3: 100k scan vs the 2M map at 1 m voxels (mode 7 / 27) vs GICP."""
    sc, mp, T_true, T0 = gen.config_c3()
    md, sd = D(mp), D(sc)
    im = g.build_index(md, 0.5)
    _, _, cm = g.knn_cov_self(im, 20, with_nbr=False)
    g.attach_cov(im, cm)
    isc = g.build_index(sd, 0.0)
    _, _, cs = g.knn_cov_self(isc, 20, with_nbr=False)
    iv = g.build_index(md, 1.0)
    ms_att, _ = timed(lambda: g.attach_voxels(iv, cm))
    res = {"attach_voxels_ms": ms_att}
    for mode in (7, 27):
        ms_l, _ = timed(lambda: g.linearize_vgicp(sd, cs, iv, T_true, mode, pivot=T_true[:3, 3]))
        ms_a, (T, info) = timed(lambda: g.align_vgicp(sd, cs, iv, T0, mode), reps=3)
        res[f"mode{mode}"] = {"linearize_ms": ms_l, "align_ms": ms_a, "iterations": info.iterations,
                              "converged": info.converged, "t_err_m": float(np.linalg.norm(T[:3, 3] - T_true[:3, 3]))}
    ms_l, _ = timed(lambda: g.linearize(sd, cs, im, cm, T_true, 1.0, pivot=T_true[:3, 3]))
    ms_a, (T, info) = timed(lambda: g.align(sd, cs, im, cm, T0), reps=3)
    res["gicp"] = {"linearize_ms": ms_l, "align_ms": ms_a, "iterations": info.iterations,
                   "t_err_m": float(np.linalg.norm(T[:3, 3] - T_true[:3, 3]))}
    print(json.dumps({"workload": "VGICP vs GICP, C3 100k scan vs 2M map (voxel 1.0 m)", **res}))


def gc():
    """z-vote ground filter + Euclidean clustering on the C3 scan (vehicle frame)."""
    sc, _ = gen.scan(100_000, gen.C3_U, 1000)
    _, first = np.unique(np.floor(sc / 0.25).astype(np.int64), axis=0, return_index=True)
    vf = np.ascontiguousarray(sc[np.sort(first)])
    sd = D(vf)
    ms_g, keep = timed(lambda: g.ground_filter(sd, 0.5, 6))
    feat = sd[keep].contiguous()
    ms_c, (lab, nc) = timed(lambda: g.cluster(feat, 0.5, 10))
    print(json.dumps({"workload": "ground filter + clustering, C3 scan voxel-filtered at 0.25 m",
                      "points": int(sd.shape[0]), "kept": int(feat.shape[0]), "ground_filter_ms": ms_g,
                      "cluster_ms": ms_c, "clusters": nc}))


if __name__ == "__main__":
    args = sys.argv[1:] or ["c2", "c4", "c5"]
    i = 0
    while i < len(args):
        a = args[i]
        if a == "c2":
            c2()
        elif a == "c4":
            B = 16
            if i + 1 < len(args) and args[i + 1].isdigit():
                B = int(args[i + 1])
                i += 1
            c4(B)
        elif a == "c5":
            c5()
        elif a == "kd":
            kd()
        elif a == "vg":
            vg()
        elif a == "gc":
            gc()
        i += 1
