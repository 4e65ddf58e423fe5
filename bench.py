#!/usr/bin/env python
"""bench.py -- the GICP hot path on B200 (BASELINE.json metric; workload C4 by default).

Default workload (--workload c4, BASELINE.json configs[3], the north star's "batched
scan registration" across GPUs): B = 256 scan-to-map registrations -- 32 distinct
100k-point 3-LiDAR scans (C4 scans 0, 8, ..., 248: seeds 1000 + i at arc length
i L / 256) x 8 initial-pose hypotheses each (the perturbations of C4 registrations
8j .. 8j+7) -- against the shared 2M-point racetrack map, k = 20, GICP to convergence.

One STEP = the whole hot path for the batch:
  A1-A3 map   voxel index + fused kNN(k=20)+covariance of every map point
              (replicated on every rank: the map is shared),
  (scans      one NCCL all_gather of the distinct scans' points: rank r holds its
              32/N scans, every rank needs its chunks of every registration)
  A1-A3 scans index + kNN(k=20)+covariance of the distinct scans (scan-sharded:
              rank r its 32/N scans) + one NCCL all_gather of their covariances,
  A4-A7       the 256 registrations' lockstep LM with every registration's points
              split over the ranks by a fixed global chunking: per evaluation round
              one batched linearisation launch, ONE NCCL all_reduce of the device
              chunk table, the chunk-ordered combine on the device
              (gicp_align_batched_sharded), the host LM.
value    = registered scan points / step time (256 x 100k per step), inputs resident
           in HBM, L2 flushed (256 MiB write) before every timed step, max over ranks.
e2e      = the same through the public API from pinned HOST buffers (H2D of the map
           and this rank's scans inside the timed region, D2H of the 256 poses).
roofline = the step's dominant kernel (the batched linearisation; 80 B per source
           point per launch); roofline_knn_cov = the map's fused
           kNN+covariance (304 B/point at k = 20), the north star's 1-GPU target.
--impl reference times the oracle (CPU, this box's cores) on a bounded sample of
the same workload: one registration's seeded 2000-point subsample, its covariance
inputs and the map cropped exactly around it, kNN+covariance + LM to convergence.

--workload c3 keeps the round-1 step (one 100k scan vs the 2M map, map index +
kNN/cov + scan + align; N > 1: replicas) for comparison.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

K = 20
EPS = 1e-3
LIN_BYTES_PER_PT = 80   # linearize, per source point per launch
MAP_CELL = 0.5          # m, ~1.15 x the 20-NN radius at 31 pts/m^2
METRIC = "kNN+covariance points/sec (k=20) and GICP iters/sec; % HBM roofline"
BYTES_PER_PT = 64 + 12 * K   # kNN+cov, queries = cloud
N_DISTINCT, N_HYP = 32, 8    # C4: 32 distinct scans x 8 initial poses = 256 registrations
N_SCAN = 100_000
WORKLOAD_C4 = ("C4 batched scan-to-map: 256 registrations (32 distinct 100k-point 3-LiDAR scans x 8 initial-pose "
               "hypotheses) vs the shared 2M-point racetrack map, k=20, GICP to convergence, source points "
               "sharded over the GPUs (NCCL chunk-table allreduce per round)")
WORKLOAD_C3 = "C3 scan-to-map: 100k-point scan vs 2M-point racetrack map, k=20, GICP to convergence"
REF_SUB = 2000               # oracle sample: source points of one registration
ALIGN_GROUPS = int(os.environ.get("BENCH_ALIGN_GROUPS", "4"))   # concurrent batched aligns (sharding.ConcurrentAlign)
SCAN_WORKERS = int(os.environ.get("BENCH_SCAN_WORKERS", "8"))   # host threads issuing the scans' kNN/cov


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self, t0=None, t1=None):
        """Samples received during [t0, t1] (host clock; the whole run if None)."""
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ts, ln in self.lines:
            if t0 is not None and not (t0 <= ts <= t1):
                continue
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nme, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nme)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------------------
# the C4 batch (shared by both arms)
# ------------------------------------------------------------------------------

def _gen_scan(j):
    import gen
    sc, T, _ = gen.config_c4_scan(N_HYP * j, N_SCAN)
    return np.ascontiguousarray(sc), T


def c4_poses():
    """T0 of registration b = 8j + h: scan j's T_true composed with the perturbation of
    C4 registration b (gen.config_c4_scan's recipe), and the T_true of each scan."""
    import gen
    Tt, T0 = [], []
    for j in range(N_DISTINCT):
        u = N_HYP * j * gen.TRACK_LEN / 256.0
        T = gen.vehicle_pose(u)
        Tt.append(T)
        for h in range(N_HYP):
            b = N_HYP * j + h
            T0.append(T @ gen.perturbation(0.5, 1.0, 1000 + b + 7))
    return np.array(Tt), np.array(T0)


def gen_scans(js, workers):
    """The distinct scans js (process pool: the generator is numpy-bound)."""
    if workers <= 1 or len(js) <= 1:
        return [_gen_scan(j) for j in js]
    from concurrent.futures import ProcessPoolExecutor
    import multiprocessing as mp
    with ProcessPoolExecutor(max_workers=workers, mp_context=mp.get_context("fork")) as ex:
        return list(ex.map(_gen_scan, js))


# ------------------------------------------------------------------------------
# reference arm: the oracle on the host cores
# ------------------------------------------------------------------------------

def oracle_registration_sample(seed: int):
    """The oracle on a bounded sample of the C4 workload: registration b = 8 j + h
    (seeded), a seeded REF_SUB-point subsample of its scan, the map cropped EXACTLY to
    the subsample's bounding box at T0 plus 4 m (a map point outside can only be a
    correspondence after a move of > 3 m; kept in original order), the covariance
    inputs by the oracle's kNN(k=20)+covariance (source points against the full scan,
    crop points against the crop + 1.5 m), then O4 to convergence. Returns
    (points/s, seconds, iterations)."""
    import gen
    import oracle
    oracle.build()
    rng = np.random.default_rng(seed)
    j = int(rng.integers(N_DISTINCT))
    h = int(rng.integers(N_HYP))
    sc, _ = _gen_scan(j)
    _, T0s = c4_poses()
    T0 = T0s[N_HYP * j + h]
    mp = gen.racetrack_map(2_000_000, 1)
    t0 = time.perf_counter()
    sub = np.sort(rng.choice(len(sc), REF_SUB, replace=False))
    src = np.ascontiguousarray(sc[sub])
    pw = src.astype(np.float64) @ T0[:3, :3].T + T0[:3, 3]
    lo, hi = pw.min(0) - 4.0, pw.max(0) + 4.0
    inb = np.all((mp >= lo) & (mp <= hi), axis=1)
    inb2 = np.all((mp >= lo - 1.5) & (mp <= hi + 1.5), axis=1)
    crop, crop2 = np.ascontiguousarray(mp[inb]), np.ascontiguousarray(mp[inb2])
    nb_c, _ = oracle.knn(crop2, crop, K)
    ct = oracle.covariance(crop2, nb_c, EPS)[0].astype(np.float32)
    nb_s, _ = oracle.knn(sc, src, K)
    cs = oracle.covariance(sc, nb_s, EPS)[0].astype(np.float32)
    r = oracle.align(src, cs, crop, ct, T0)
    dt = time.perf_counter() - t0
    return REF_SUB / dt, dt, r["iterations"]


def reference_main(args, rank, world):
    if rank != 0:
        return 0
    cores = os.cpu_count() or 1
    for w in range(min(args.warmup, 1)):
        oracle_registration_sample(900 + w)
    vals, secs, its = [], [], []
    for s in range(args.steps):
        v, dt, it = oracle_registration_sample(77 + s)
        vals.append(v)
        secs.append(dt)
        its.append(it)
    v = statistics.mean(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "registered scan points/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(secs),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32/f64",
        "data": "synthetic racetrack (gen/, seeded)",
        "config": {"workload": WORKLOAD_C4, "k": K, "map_points": 2_000_000, "scan_points": N_SCAN,
                   "registrations": N_DISTINCT * N_HYP, "l2": "n/a (CPU)"},
        "cpu_baseline": {"value": v, "unit": "registered scan points/s", "cores": cores, "kind": "oracle",
                         "sample": f"per step one seeded registration: a {REF_SUB}-point subsample of its scan, "
                                   f"covariance inputs (oracle kNN+cov) and O4 to convergence against the map "
                                   f"cropped exactly around it (mean {statistics.mean(its):.1f} iterations); "
                                   f"ms_per_step is the measured time of that sample"},
        "e2e": {"value": v, "unit": "registered scan points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------
# our arm, C4 (default)
# ------------------------------------------------------------------------------

def masked_fraction(xyz, nbr, rows=20000, seed=5):
    """SURVEY §8 tolerances: the fraction of kNN rows whose neighbour set is nearly
    degenerate (eigen-gap (l1 - l0) / l2 of its covariance below 1e-2), where the
    covariance check falls back to properties. Measured outside the timed region on
    a seeded sample of the GPU's rows (numpy eigvalsh; a report, not the product)."""
    nb = nbr.cpu().numpy() if hasattr(nbr, "cpu") else np.asarray(nbr)
    sel = np.random.default_rng(seed).choice(nb.shape[0], min(rows, nb.shape[0]), replace=False)
    P = np.asarray(xyz, np.float64)[nb[sel]]
    D = P - P.mean(axis=1, keepdims=True)
    lam = np.linalg.eigvalsh(np.einsum("rki,rkj->rij", D, D) / P.shape[1])
    gap = np.where(lam[:, 2] > 0, (lam[:, 1] - lam[:, 0]) / np.where(lam[:, 2] > 0, lam[:, 2], 1.0), 0.0)
    return {"value": float((gap < 1e-2).mean()), "gap_below": 1e-2, "rows_sampled": int(len(sel)),
            "of": f"the 2M map's k={nb.shape[1]} rows", "bar": 0.01}


def run_c4(args, rank, world, local):
    import torch
    import torch.distributed as dist

    import gen
    import paper_2308_07173_b200 as g
    from paper_2308_07173_b200 import sharding

    if N_DISTINCT % world:
        raise SystemExit(f"--gpus must divide {N_DISTINCT}")
    per = N_DISTINCT // world
    mine = list(range(rank * per, (rank + 1) * per))
    B = N_DISTINCT * N_HYP
    # --- inputs (host generation before any CUDA work: the pool forks) ---
    scans = gen_scans(mine, max(1, min(len(mine), (os.cpu_count() or 1) // world)))
    mp = gen.racetrack_map(2_000_000, 1)

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    T_true, T0 = c4_poses()
    map_d = torch.from_numpy(mp).to(dev)
    my_scans = torch.from_numpy(np.concatenate([s for s, _ in scans])).to(dev)   # [per * N_SCAN, 3]
    all_scans = torch.empty((N_DISTINCT * N_SCAN, 3), dtype=torch.float32, device=dev)
    cov_mine = torch.empty((per * N_SCAN, 6), dtype=torch.float32, device=dev)
    cov_all = torch.empty((N_DISTINCT * N_SCAN, 6), dtype=torch.float32, device=dev)
    offsets = np.arange(B + 1, dtype=np.int64) * N_SCAN
    reg_base = (np.arange(B) // N_HYP) * N_SCAN                          # registration b -> its scan's rows
    plan = sharding.ShardPlan(offsets, dev, num_chunks=sharding.NUM_CHUNKS, reg_base=reg_base)
    # the timed steps align the batch as ALIGN_GROUPS concurrent groups (each its own
    # host thread + stream: one group's kernels fill the GPU while another's host LM
    # takes its round decision); results are bitwise those of the single call
    conc = sharding.ConcurrentAlign(offsets, dev, ALIGN_GROUPS, num_chunks=sharding.NUM_CHUNKS, reg_base=reg_base)
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    from concurrent.futures import ThreadPoolExecutor
    side = [torch.cuda.Stream(device=dev) for _ in range(SCAN_WORKERS)]
    pool = ThreadPoolExecutor(max_workers=SCAN_WORKERS, initializer=lambda: torch.cuda.set_device(local))

    def step(map_src, scan_src, record=None, single=False):
        e = [ev() for _ in range(5)]
        e[0].record(stream)
        if world > 1:                              # every rank needs every scan's points (its chunks)
            dist.all_gather_into_tensor(all_scans, scan_src)
        else:
            all_scans.copy_(scan_src)
        imap = g.build_index(map_src, MAP_CELL)
        _, _, cov_map = g.knn_cov_self(imap, K, EPS, with_nbr=True)
        g.attach_cov(imap, cov_map)
        e[1].record(stream)
        # the distinct scans' index + kNN/cov: latency-bound small clouds (host-synchronising
        # index builds), so SCAN_WORKERS host threads run them on their own streams at once
        start = torch.cuda.Event()
        start.record(stream)

        def scan_job(w):
            sw = side[w]
            sw.wait_event(start)
            with torch.cuda.stream(sw):
                for i in range(w, per, SCAN_WORKERS):
                    sl = scan_src[i * N_SCAN:(i + 1) * N_SCAN]
                    isc = g.build_index(sl, 0.0)
                    g.knn_cov_self(isc, K, EPS, with_nbr=True, out=(None, None, cov_mine[i * N_SCAN:(i + 1) * N_SCAN]))
                    isc.free()
            done = torch.cuda.Event()
            done.record(sw)
            return done
        for d in list(pool.map(scan_job, range(SCAN_WORKERS))):
            stream.wait_event(d)
        if world > 1:
            dist.all_gather_into_tensor(cov_all, cov_mine)
        else:
            cov_all.copy_(cov_mine)
        e[2].record(stream)
        if single or ALIGN_GROUPS <= 1:
            T, infos = sharding.align_batched_sharded(g, all_scans, cov_all, offsets, imap, cov_map, T0, plan=plan)
        else:
            T, infos = conc(g, all_scans, cov_all, imap, cov_map, T0)
        e[3].record(stream)
        if record is not None:
            record.append((e, infos, T))
        imap.free()
        return T, infos

    with ClockSampler(local) as clk:
        for _ in range(args.warmup):
            step(map_d, my_scans)
        torch.cuda.synchronize()
        time.sleep(0.3)
        rec, step_ms = [], []
        t_start = time.time()
        for si in range(args.steps):
            flush.zero_()                          # L2 flush (256 MiB > 126 MB L2), outside the timed region
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            t0, t1 = ev(), ev()
            t0.record(stream)
            step(map_d, my_scans, rec)
            t1.record(stream)
            torch.cuda.synchronize()
            step_ms.append(t0.elapsed_time(t1))
        t_end = time.time()
        time.sleep(0.15)
    clocks = clk.summary(t_start, t_end + 0.1)
    # the dominant kernel's roofline: per-launch events over one extra, untimed step run
    # as a single batched call (concurrent groups would share the GPU inside each
    # launch's event window)
    flush.zero_()
    torch.cuda.synchronize()
    g.align_timing(True)
    step(map_d, my_scans, None, single=True)
    torch.cuda.synchronize()
    lin_ms, lin_n, lin_pts = g.align_timing(False)

    def maxr(x):
        if world == 1:
            return x
        t = torch.tensor([x], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    ms = maxr(statistics.mean(step_ms))
    map_ms = statistics.mean(r[0][0].elapsed_time(r[0][1]) for r in rec)
    scan_ms = statistics.mean(r[0][1].elapsed_time(r[0][2]) for r in rec)
    align_ms = statistics.mean(r[0][2].elapsed_time(r[0][3]) for r in rec)
    infos = rec[-1][1]
    iters = sum(i.iterations for i in infos)
    T_last = rec[-1][2]
    errs = [float(np.linalg.norm(T_last[b][:3, 3] - T_true[b // N_HYP][:3, 3])) for b in range(B)]
    value = B * N_SCAN / (ms * 1e-3)
    peak, peak_kind = peaks()

    # the map's kNN+cov alone (the north star's 1-GPU target), CUDA events, L2 flushed
    imap = g.build_index(map_d, MAP_CELL)
    kn = []
    for _ in range(6):
        flush.zero_()
        a, b = ev(), ev()
        a.record(stream)
        nbr_map, _, _ = g.knn_cov_self(imap, K, EPS, with_nbr=True)
        b.record(stream)
        torch.cuda.synchronize()
        kn.append(a.elapsed_time(b))
    imap.free()
    masked = masked_fraction(mp, nbr_map)
    knn_ms = statistics.median(kn[1:])
    knn_ach = mp.shape[0] * BYTES_PER_PT / (knn_ms * 1e-3) / 1e9
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    traffic = json.load(open(tp)) if os.path.exists(tp) else {}
    roof_knn = {"bound": "hbm", "achieved": knn_ach, "peak": peak, "unit": "GB/s", "frac": knn_ach / peak,
                "traffic": traffic.get("k_knn_self_map_bytes_per_launch"), "peak_kind": peak_kind,
                "kernel": "gicp_knn_cov_self on the 2M map (tiled stage + per-query fallback, escalation, exact)",
                "bytes_per_point": BYTES_PER_PT, "ms": knn_ms,
                "timed": "alone, CUDA events around the call, L2 flushed, median of 5"}
    # the batched linearisation: algorithmic bytes of the launches' active points
    lin_all_ms = sum(lin_ms)
    roof_lin = None
    if lin_n[0]:
        ach = LIN_BYTES_PER_PT * lin_pts[0] / (lin_ms[0] * 1e-3) / 1e9
        roof_lin = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                    "traffic": traffic.get("k_linearize_batched_bytes_per_launch"), "peak_kind": peak_kind,
                    "kernel": "k_linearize (batched speculative dual launch, gicp_align_batched_sharded)",
                    "bytes_per_point": LIN_BYTES_PER_PT, "points_per_launch": lin_pts[0] / lin_n[0],
                    "launch_ms": lin_ms[0] / lin_n[0], "launches_per_step": sum(lin_n),
                    "linearize_ms_per_step": lin_all_ms,
                    "timed": "CUDA events around every linearisation launch of one extra untimed step run as a single batched call (the timed steps align ALIGN_GROUPS concurrent groups)"}

    # --- launches per step (CUPTI via torch.profiler, one extra untimed step) ---
    gpu_launches = None
    try:
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            step(map_d, my_scans)
            torch.cuda.synchronize()
        names = [e.name for e in prof.events() if e.device_type.name == "CUDA"]
        ours = [n for n in names if ("gicp" in n or "cub" in n.lower())]
        gpu_launches = len(ours) * args.steps
    except Exception:
        gpu_launches = None

    # --- e2e: the same step through the public API from pinned host buffers ---
    e2e = None
    if not args.no_e2e:
        map_h = torch.from_numpy(mp).pin_memory()
        scan_h = my_scans.cpu().pin_memory()
        pose_h = torch.empty((B, 16), dtype=torch.float64).pin_memory()
        em = []
        for it in range(max(2, args.steps // 4) + 1):
            flush.zero_()
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            a, b = ev(), ev()
            a.record(stream)
            md = map_h.to(dev, non_blocking=True)
            sd = scan_h.to(dev, non_blocking=True)
            T, _ = step(md, sd)
            pose_h.copy_(torch.from_numpy(np.asarray(T).reshape(B, 16)))   # the poses come back to the host
            b.record(stream)
            torch.cuda.synchronize()
            if it > 0:
                em.append(a.elapsed_time(b))
        e2e_ms = maxr(statistics.mean(em))
        e2e = {"value": B * N_SCAN / (e2e_ms * 1e-3), "unit": "registered scan points/s",
               "h2d_bytes_per_step": int(mp.nbytes + scan_h.numel() * 4), "d2h_bytes_per_step": int(B * 16 * 8),
               "ms_per_step": e2e_ms}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, dt, it = oracle_registration_sample(77)
        cpu = {"value": v, "unit": "registered scan points/s", "cores": os.cpu_count(), "kind": "oracle",
               "sample": f"one seeded registration: a {REF_SUB}-point subsample, its covariance inputs (oracle "
                         f"kNN+cov) and O4 to convergence ({it} iterations) against the map cropped exactly "
                         f"around it, {dt:.1f} s"}

    if rank == 0:
        dominant = roof_lin if (roof_lin is not None and lin_all_ms >= knn_ms) else roof_knn
        line = {
            "metric": METRIC, "value": value, "unit": "registered scan points/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32 (kNN/cov, per-point terms), f64 (transform, reductions, LM)",
            "data": "synthetic racetrack (gen/, seeded): 2M-point map, 32 distinct 100k-point 3-LiDAR scans",
            "config": {"workload": WORKLOAD_C4, "k": K, "map_points": int(mp.shape[0]), "scan_points": N_SCAN,
                       "registrations": B, "distinct_scans": N_DISTINCT, "map_cell_m": MAP_CELL,
                       "l2": "flushed (256 MiB write) before every timed step",
                       "parallelism": f"points of every registration sharded over {world} GPU(s) "
                                      f"({sharding.NUM_CHUNKS} fixed chunks, NCCL chunk-table allreduce per round); "
                                      f"distinct scans sharded for kNN+cov (NCCL all_gather); map replicated; "
                                      f"the batch aligned as {ALIGN_GROUPS} concurrent groups per GPU (host threads + "
                                      f"streams, round-robin ordered collectives)"},
            "gicp_iters_per_s": iters / (align_ms * 1e-3),
            "knn_cov_points_per_s": mp.shape[0] / (knn_ms * 1e-3),
            "breakdown_ms": {"map_index_knn_cov": map_ms, "scan_index_knn_cov_allgather": scan_ms,
                             "batched_align": align_ms, "iterations_total": iters,
                             "iterations_mean": iters / B},
            "align_translation_error_m": {"median": float(np.median(errs)), "max": float(np.max(errs))},
            "roofline": dominant,
            "masked_fraction": masked,
            "roofline_knn_cov": roof_knn,
            "roofline_linearize": roof_lin,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": gpu_launches,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


# ------------------------------------------------------------------------------
# our arm, C3 (round 1's step; --workload c3)
# ------------------------------------------------------------------------------

def run_c3(args, rank, world, local):
    import torch
    import torch.distributed as dist

    import gen
    import paper_2308_07173_b200 as g

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    sc, mp, T_true, T0 = gen.config_c3(scan_seed=1000 + rank)
    map_d = torch.from_numpy(np.array(mp)).to(dev)
    scan_d = torch.from_numpy(np.array(sc)).to(dev)
    n_pts = mp.shape[0] + sc.shape[0]
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    sb = torch.cuda.Stream(device=dev, priority=-1)
    from concurrent.futures import ThreadPoolExecutor
    pool = ThreadPoolExecutor(max_workers=1, initializer=lambda: torch.cuda.set_device(local))

    def scan_path(e, after):
        sb.wait_event(after)
        with torch.cuda.stream(sb):
            e[5].record(sb)
            iscan = g.build_index(scan_d, 0.0)
            _, _, cov_scan = g.knn_cov_self(iscan, K, EPS, with_nbr=True)
            e[3].record(sb)
        return iscan, cov_scan

    def step(record=None):
        e = [ev() for _ in range(6)]
        e[0].record(stream)
        fut = pool.submit(scan_path, e, e[0])
        imap = g.build_index(map_d, MAP_CELL)
        e[1].record(stream)
        _, _, cov_map = g.knn_cov_self(imap, K, EPS, with_nbr=True)
        g.attach_cov(imap, cov_map)
        e[2].record(stream)
        iscan, cov_scan = fut.result()
        stream.wait_stream(sb)
        cov_scan.record_stream(stream)
        T, info = g.align(scan_d, cov_scan, imap, cov_map, T0)
        e[4].record(stream)
        if record is not None:
            record.append((e, info, T))
        imap.free()
        iscan.free()
        return T, info

    with ClockSampler(local) as clk:
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        time.sleep(0.3)
        rec, step_ms = [], []
        t_start = time.time()
        for si in range(args.steps):
            g.align_timing(si == args.steps - 1)
            flush.zero_()
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            t0, t1 = ev(), ev()
            t0.record(stream)
            step(rec)
            t1.record(stream)
            torch.cuda.synchronize()
            step_ms.append(t0.elapsed_time(t1))
        lin_ms, lin_n, lin_pts = g.align_timing(False)
        t_end = time.time()
        time.sleep(0.15)
    clocks = clk.summary(t_start, t_end + 0.1)
    ms = statistics.mean(step_ms)
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    build_ms = statistics.mean(r[0][0].elapsed_time(r[0][1]) for r in rec)
    knncov_ms = statistics.mean(r[0][1].elapsed_time(r[0][2]) for r in rec)
    scan_ms = statistics.mean(r[0][5].elapsed_time(r[0][3]) for r in rec)
    align_ms = statistics.mean(r[0][0].elapsed_time(r[0][4]) - max(r[0][0].elapsed_time(r[0][2]),
                                                                    r[0][0].elapsed_time(r[0][3])) for r in rec)
    iters = statistics.mean(r[1].iterations for r in rec)
    peak, peak_kind = peaks()
    achieved = mp.shape[0] * BYTES_PER_PT / (knncov_ms * 1e-3) / 1e9
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": None, "peak_kind": peak_kind, "kernel": "gicp_knn_cov_self on the 2M map (in the step)",
            "bytes_per_point": BYTES_PER_PT, "ms_per_step": knncov_ms}
    roof_lin = None
    if lin_n[0]:
        ach = LIN_BYTES_PER_PT * lin_pts[0] / (lin_ms[0] * 1e-3) / 1e9
        roof_lin = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                    "traffic": None, "peak_kind": peak_kind, "kernel": "k_linearize (speculative dual launch)",
                    "bytes_per_point": LIN_BYTES_PER_PT, "launch_ms": lin_ms[0] / lin_n[0],
                    "launches_per_step": sum(lin_n), "ms_per_step": sum(lin_ms)}
    if rank == 0:
        line = {
            "metric": METRIC, "value": world * n_pts / (ms * 1e-3), "unit": "points/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32 (kNN/cov), f64 (transform, reductions, LM)",
            "data": "synthetic racetrack (gen/, seeded): 2M-point map, 100k-point 3-LiDAR scan",
            "config": {"workload": WORKLOAD_C3, "k": K, "map_points": int(mp.shape[0]),
                       "scan_points": int(sc.shape[0]), "map_cell_m": MAP_CELL,
                       "l2": "flushed (256 MiB write) before every timed step", "parallelism": f"replicas x{world}"},
            "gicp_iters_per_s": iters / (align_ms * 1e-3),
            "breakdown_ms": {"map_index_build": build_ms, "map_knn_cov": knncov_ms, "scan_index_knn_cov": scan_ms,
                             "align": align_ms, "align_iterations": iters},
            "align_translation_error_m": float(np.linalg.norm(rec[-1][2][:3, 3] - T_true[:3, 3])),
            "roofline": roof if (roof_lin is None or knncov_ms >= sum(lin_ms)) else roof_lin,
            "roofline_knn_cov": roof, "roofline_linearize": roof_lin, "cpu_baseline": None, "e2e": None,
            "gpu_launches": None, "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c4", choices=["c4", "c3"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return reference_main(args, rank, world)
    if args.workload == "c3":
        return run_c3(args, rank, world, local)
    return run_c4(args, rank, world, local)


if __name__ == "__main__":
    sys.exit(main())
