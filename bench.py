#!/usr/bin/env python
"""bench.py -- the GICP hot path on B200 (BASELINE.json metric, config C3).

One STEP = one pass of the whole hot path on the C3
scan-to-map workload: build the voxel index of the 2M-point racetrack map, fused
kNN(k=20)+covariance of every map point, index + kNN+covariance of the 100k-point
scan, and GICP alignment of the scan to the map to convergence (linearize on the
GPU, LM on the host).

value  = (map + scan points through kNN+covariance) / step time  [points/s], inputs
         resident in HBM, L2 flushed (256 MiB write) before every timed step.
e2e    = the same through the public API from pinned HOST buffers: H2D of map and
         scan, the step, D2H of the map/scan covariances and the pose.
roofline = the fused kNN+covariance kernel on the map: algorithmic bytes
         (64 + 12k B/point) / its CUDA-event time.
--impl reference times the oracle (CPU, this box's cores) on a bounded sample.

Multi-GPU (torchrun): weak scaling -- every rank runs its own C3 instance (map
replicated, its own scan seed); no data-path collective.
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
LIN_BYTES_PER_PT = 80   # linearize, per source point per iteration
MAP_CELL = 0.5          # m, ~1.15 x the 20-NN radius at 31 pts/m^2
METRIC = "kNN+covariance points/sec (k=20) and GICP iters/sec; % HBM roofline"
WORKLOAD = "C3 scan-to-map: 100k-point scan vs 2M-point racetrack map, k=20, GICP to convergence"
BYTES_PER_PT = 64 + 12 * K   # kNN+cov, queries = cloud


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
# reference arm: the oracle on the host cores
# ------------------------------------------------------------------------------

def run_oracle_sample(n_queries: int, seed: int = 77):
    """kNN(k=20)+covariance of a fixed sample of map points against the FULL 2M map
    with the oracle (brute force, all host cores). Returns (points/s, seconds)."""
    import gen
    import oracle
    oracle.build()
    _, mp, _, _ = gen.config_c3()
    rng = np.random.default_rng(seed)
    rows = rng.choice(len(mp), n_queries, replace=False)
    t0 = time.perf_counter()
    nbr, _ = oracle.knn(mp, mp[rows], K)
    oracle.covariance(mp, nbr, EPS)
    dt = time.perf_counter() - t0
    return n_queries / dt, dt


def reference_main(args, rank, world):
    if rank != 0:
        return 0
    cores = os.cpu_count() or 1
    n_q = args.ref_queries
    vals = []
    for _ in range(min(args.warmup, 1)):
        run_oracle_sample(max(16, n_q // 16))
    for s in range(args.steps):
        v, dt = run_oracle_sample(n_q, seed=77 + s)
        vals.append(v)
    v = statistics.mean(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "points/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * (2_100_000 / v),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32/f64",
        "data": "synthetic racetrack (gen/, seeded)",
        "config": {"workload": WORKLOAD, "k": K, "map_points": 2_000_000, "scan_points": 100_000,
                   "l2": "n/a (CPU)"},
        "cpu_baseline": {"value": v, "unit": "points/s", "cores": cores, "kind": "oracle",
                         "sample": f"{n_q} map points (seeded) kNN(k=20)+covariance vs the full 2M map, brute force; "
                                   f"ms_per_step extrapolated to 2.1M points"},
        "e2e": {"value": v, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------
# our arm
# ------------------------------------------------------------------------------

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-queries", type=int, default=20000, help="oracle sample per reference step")
    ap.add_argument("--cpu-queries", type=int, default=60000, help="oracle sample for cpu_baseline (~10 s)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return reference_main(args, rank, world)

    import torch
    import torch.distributed as dist

    import gen
    import paper_2308_07173_b200 as g

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    # --- inputs (resident in HBM) ---
    scan_seed = 1000 + rank
    sc, mp, T_true, T0 = gen.config_c3(scan_seed=scan_seed)
    map_d = torch.from_numpy(mp).to(dev)
    scan_d = torch.from_numpy(sc).to(dev)
    n_pts = mp.shape[0] + sc.shape[0]
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    # the scan's path (index + kNN/covariances, latency-bound small grids) runs on a
    # high-priority side stream inside the map's kNN (throughput-bound, 15.6k blocks):
    # its blocks take SM slots as the map's retire, so it costs its share of the
    # machine, not its latency. The alignment joins both.
    sb = torch.cuda.Stream(device=dev, priority=-1)
    # BENCH_SCAN_THREAD=1 (default): a host worker thread issues the scan's path from
    # the step's start, so its index build (host-synchronising: bbox, level counts)
    # overlaps the map's index build instead of following it. The library's host
    # state is thread-local and its allocations stream-ordered; ctypes drops the GIL.
    scan_thread = os.environ.get("BENCH_SCAN_THREAD", "1") == "1"
    pool = None
    if scan_thread:
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
        fut = pool.submit(scan_path, e, e[0]) if scan_thread else None
        imap = g.build_index(map_d, MAP_CELL)
        e[1].record(stream)
        _, _, cov_map = g.knn_cov_self(imap, K, EPS, with_nbr=True)
        g.attach_cov(imap, cov_map)
        e[2].record(stream)
        iscan, cov_scan = fut.result() if scan_thread else scan_path(e, e[1])
        stream.wait_stream(sb)
        cov_scan.record_stream(stream)
        T, info = g.align(scan_d, cov_scan, imap, cov_map, T0)
        e[4].record(stream)
        if record is not None:
            record.append((e, info, T))
        imap.free()
        iscan.free()
        return T, info

    # warm-up (the clock sampler starts first: nvidia-smi needs ~0.1-0.5 s to come up)
    with ClockSampler(local) as clk:
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        time.sleep(0.3)
        rec = []
        step_ms = []
        t_start = time.time()
        for si in range(args.steps):
            # per-launch CUDA events around gicp_align's linearisations during the last
            # timed step only (the event records would otherwise add ~4 % to every step)
            g.align_timing(si == args.steps - 1)
            flush.zero_()  # L2 flush (256 MiB > 126 MB L2), outside the timed region
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            t0 = ev()
            t1 = ev()
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
    # the scan path overlaps the map's index build and kNN: scan_ms from its own start
    # to its own end; align from the later of the two ends
    scan_ms = statistics.mean(r[0][5].elapsed_time(r[0][3]) for r in rec)
    align_ms = statistics.mean(r[0][0].elapsed_time(r[0][4]) - max(r[0][0].elapsed_time(r[0][2]),
                                                                    r[0][0].elapsed_time(r[0][3])) for r in rec)
    iters = statistics.mean(r[1].iterations for r in rec)
    T_last = rec[-1][2]
    dt_err = float(np.linalg.norm(T_last[:3, 3] - T_true[:3, 3]))

    value = world * n_pts / (ms * 1e-3)
    peak, peak_kind = peaks()
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    achieved = mp.shape[0] * BYTES_PER_PT / (knncov_ms * 1e-3) / 1e9
    # the linearisation (the step's largest kernel share: 26 launches per step):
    # algorithmic bytes per source point per launch = 12 xyz + 24 cov
    # + 40 target float4 + cov + 4 corr = 80 B; average launch time from the events
    lin_bytes = LIN_BYTES_PER_PT * lin_pts
    lin_launch_ms = lin_ms[0] / max(lin_n[0], 1)
    lin_achieved = lin_bytes / (lin_launch_ms * 1e-3) / 1e9 if lin_n[0] else None
    lin_step_ms = sum(lin_ms)  # one step's worth (the last timed step)
    lin_traffic = None
    if os.path.exists(tp):
        try:
            lin_traffic = json.load(open(tp)).get("k_linearize_dual_bytes_per_launch")
        except Exception:
            lin_traffic = None
    traffic = None
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get("k_knn_self_map_bytes_per_launch")
        except Exception:
            traffic = None

    # --- launches per step (CUPTI via torch.profiler, one extra untimed step) ---
    gpu_launches = None
    try:
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            step()
            torch.cuda.synchronize()
        names = [e.name for e in prof.events() if e.device_type.name == "CUDA"]
        ours = [n for n in names if ("gicp" in n or "cub" in n.lower())]
        gpu_launches = len(ours) * args.steps
    except Exception:
        gpu_launches = None

    # --- e2e through the public API from pinned host buffers ---
    e2e = None
    if not args.no_e2e:
        map_h = torch.from_numpy(mp).pin_memory()
        scan_h = torch.from_numpy(sc).pin_memory()
        cov_map_h = torch.empty((mp.shape[0], 6), dtype=torch.float32).pin_memory()
        cov_scan_h = torch.empty((sc.shape[0], 6), dtype=torch.float32).pin_memory()
        e2e_ms = []
        # transfers overlap the compute on a copy stream: the scan goes up first and
        # its index + kNN/covariances run while the map uploads; the map covariances'
        # download overlaps the alignment. Both are non-default streams (the legacy
        # default stream would serialise them).
        cp = torch.cuda.Stream(device=dev)
        es = torch.cuda.Stream(device=dev)
        for it in range(args.steps + 1):
            flush.zero_()
            torch.cuda.synchronize()
            with torch.cuda.stream(es):
                a, b = ev(), ev()
                a.record(es)
                cp.wait_stream(es)
                sd = scan_h.to(dev, non_blocking=True)
                with torch.cuda.stream(cp):
                    md = map_h.to(dev, non_blocking=True)
                    up = torch.cuda.Event()
                    up.record(cp)
                iscan = g.build_index(sd, 0.0)
                _, _, cs = g.knn_cov_self(iscan, K, EPS, with_nbr=True)
                es.wait_event(up)  # the map's upload
                md.record_stream(es)
                imap = g.build_index(md, MAP_CELL)
                _, _, cm = g.knn_cov_self(imap, K, EPS, with_nbr=True)
                g.attach_cov(imap, cm)
                cp.wait_stream(es)
                with torch.cuda.stream(cp):
                    cov_map_h.copy_(cm, non_blocking=True)
                T, info = g.align(sd, cs, imap, cm, T0)
                cov_scan_h.copy_(cs, non_blocking=True)
                es.wait_stream(cp)
                b.record(es)
            torch.cuda.synchronize()
            imap.free()
            iscan.free()
            if it > 0:
                e2e_ms.append(a.elapsed_time(b))
        em = statistics.mean(e2e_ms)
        if world > 1:
            t = torch.tensor([em], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            em = float(t.item())
        e2e = {"value": world * n_pts / (em * 1e-3), "unit": "points/s",
               "h2d_bytes_per_step": int(mp.nbytes + sc.nbytes),
               "d2h_bytes_per_step": int(cov_map_h.numel() * 4 + cov_scan_h.numel() * 4 + 16 * 8),
               "ms_per_step": em}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, dt = run_oracle_sample(args.cpu_queries)
        cpu = {"value": v, "unit": "points/s", "cores": os.cpu_count(), "kind": "oracle",
               "sample": f"{args.cpu_queries} seeded map points, kNN(k=20)+covariance vs the full 2M map "
                         f"(brute force), {dt:.1f} s"}

    roof_knn = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "peak_kind": peak_kind, "kernel": "k_knn_self (fused kNN+cov, map: level, escalate, exact)",
                "bytes_per_point": BYTES_PER_PT, "ms_per_step": knncov_ms}
    roof_lin = None
    if lin_achieved is not None:
        roof_lin = {"bound": "hbm", "achieved": lin_achieved, "peak": peak, "unit": "GB/s",
                    "frac": lin_achieved / peak, "traffic": lin_traffic, "peak_kind": peak_kind,
                    "kernel": "k_linearize (speculative dual launch inside gicp_align)",
                    "bytes_per_point": LIN_BYTES_PER_PT, "points": lin_pts, "launch_ms": lin_launch_ms,
                    "launches_per_step": sum(lin_n), "ms_per_step": lin_step_ms,
                    "timed": "CUDA events around every linearisation launch of the last timed step"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "points/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32 (kNN/cov), f64 (transform, reductions, LM)",
            "data": "synthetic racetrack (gen/, seeded): 2M-point map, 100k-point 3-LiDAR scan",
            "config": {"workload": WORKLOAD, "k": K, "map_points": int(mp.shape[0]),
                       "scan_points": int(sc.shape[0]), "map_cell_m": MAP_CELL,
                       "l2": "flushed (256 MiB write) before every timed step", "parallelism": f"replicas x{world}",
                       "scan_issue": "host worker thread" if scan_thread else "main thread"},
            "gicp_iters_per_s": iters / (align_ms * 1e-3),
            "breakdown_ms": {"map_index_build": build_ms, "map_knn_cov": knncov_ms,
                             "scan_index_knn_cov": scan_ms, "align": align_ms, "align_iterations": iters},
            "knn_cov_kernel_pts_per_s": mp.shape[0] / (knncov_ms * 1e-3),
            "align_translation_error_m": dt_err,
            # the kernel with the largest share of the step (per-step device time)
            "roofline": (roof_knn if knncov_ms >= lin_step_ms or lin_achieved is None else roof_lin),
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


if __name__ == "__main__":
    sys.exit(main())
