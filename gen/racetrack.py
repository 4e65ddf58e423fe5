"""Seeded synthetic inputs for the GICP hot path (SURVEY.md §8(d) "Synthetic inputs").

This module is shared by the oracle side (tests, bench's cpu_baseline leg) and the
CUDA side. It holds NONE of the method's arithmetic: no neighbour search, no
covariance, no GICP cost, no SE(3) exponential. It only draws points on surfaces
and builds rigid transforms from Euler angles so that both sides read identical
fp32 bytes.

Workload shapes follow the paper's setting: a banked racing oval with walls and a
ground plane sampled at multi-LiDAR densities ("dense
registration using 128-channel or solid-state LiDAR"; the oval/banking per SPEC.md
l.92-95, l.116; three 120-degree Luminar-class sensors).
Dimensions (400 m straights, R = 256 m turns, 18 m ribbon, 9/20 degree bank,
walls, jittered fence posts) are the recipe stated in DESIGN.md §Inputs.
"""
from __future__ import annotations

import functools
import math

import numpy as np

# ----------------------------------------------------------------------------
# track geometry
# ----------------------------------------------------------------------------
STRAIGHT = 400.0          # m, straight length along x
RADIUS = 256.0            # m, turn radius of the centreline
HALF_WIDTH = 9.0          # m, ribbon half width (18 m ribbon)
APRON = 6.0               # m, flat apron inside the inner edge
BANK_STRAIGHT = math.radians(9.0)
BANK_TURN = math.radians(20.0)
BANK_TRANSITION = 50.0    # m, linear bank transition centred on each junction
OUTER_WALL_H = 1.2
INNER_WALL_H = 1.0
POST_R = 0.1
POST_H = 4.0
POST_SPACING = 10.0
POST_JITTER = 2.0
NOISE_SIGMA = 0.01        # m, along the surface normal

TURN_LEN = math.pi * RADIUS
TRACK_LEN = 2.0 * STRAIGHT + 2.0 * TURN_LEN
# segment starts (arc length): A straight, B turn, C straight, D turn
_U_B = STRAIGHT
_U_C = STRAIGHT + TURN_LEN
_U_D = 2.0 * STRAIGHT + TURN_LEN
_JUNCTIONS = np.array([0.0, _U_B, _U_C, _U_D, TRACK_LEN])


def centreline(u):
    """Centreline position (x, y), heading h and curvature kappa at arc length u."""
    u = np.mod(np.asarray(u, dtype=np.float64), TRACK_LEN)
    x = np.empty_like(u)
    y = np.empty_like(u)
    h = np.empty_like(u)
    k = np.zeros_like(u)
    a = u < _U_B
    x[a] = -STRAIGHT / 2 + u[a]
    y[a] = -RADIUS
    h[a] = 0.0
    b = (u >= _U_B) & (u < _U_C)
    phi = -math.pi / 2 + (u[b] - _U_B) / RADIUS
    x[b] = STRAIGHT / 2 + RADIUS * np.cos(phi)
    y[b] = RADIUS * np.sin(phi)
    h[b] = phi + math.pi / 2
    k[b] = 1.0 / RADIUS
    c = (u >= _U_C) & (u < _U_D)
    x[c] = STRAIGHT / 2 - (u[c] - _U_C)
    y[c] = RADIUS
    h[c] = math.pi
    d = u >= _U_D
    phi = math.pi / 2 + (u[d] - _U_D) / RADIUS
    x[d] = -STRAIGHT / 2 + RADIUS * np.cos(phi)
    y[d] = RADIUS * np.sin(phi)
    h[d] = phi + math.pi / 2
    k[d] = 1.0 / RADIUS
    return x, y, h, k


def bank(u):
    """Bank angle: 9 deg on straights, 20 deg in turns, 50 m linear transitions."""
    u = np.mod(np.asarray(u, dtype=np.float64), TRACK_LEN)
    in_turn = ((u >= _U_B) & (u < _U_C)) | (u >= _U_D)
    beta = np.where(in_turn, BANK_TURN, BANK_STRAIGHT)
    # distance to the nearest junction, signed so that the turn side is positive
    for j in _JUNCTIONS:
        dist = u - j
        near = np.abs(dist) < BANK_TRANSITION / 2
        if not near.any():
            continue
        # junctions 0/C start a straight (turn before), B/D start a turn
        starts_turn = j in (_U_B, _U_D)
        s = dist[near] if starts_turn else -dist[near]
        frac = 0.5 + s / BANK_TRANSITION  # 0 at the straight side, 1 at the turn side
        beta[near] = BANK_STRAIGHT + (BANK_TURN - BANK_STRAIGHT) * frac
    return beta


def _frame(u):
    x, y, h, k = centreline(u)
    out = np.stack([np.sin(h), -np.cos(h)], axis=-1)  # outward (right of CCW travel)
    return x, y, h, k, out


def _surface_point(u, w, kind, rng_extra=None):
    """Point on a surface at arc length u and lateral offset w (outward positive)."""
    x, y, h, k, out = _frame(u)
    beta = bank(u)
    px = x + w * out[:, 0]
    py = y + w * out[:, 1]
    if kind == "ribbon":
        pz = (w + HALF_WIDTH) * np.tan(beta)
        # normal of z = (w+9) tan(beta): tilted toward the infield
        nx = -np.sin(beta) * out[:, 0]
        ny = -np.sin(beta) * out[:, 1]
        nz = np.cos(beta)
    elif kind == "apron":
        pz = np.zeros_like(u)
        nx, ny, nz = np.zeros_like(u), np.zeros_like(u), np.ones_like(u)
    else:
        raise ValueError(kind)
    return np.stack([px, py, pz], -1), np.stack([nx, ny, nz], -1)


# ----------------------------------------------------------------------------
# surface samplers (all vectorised, seeded)
# ----------------------------------------------------------------------------

def _sample_strip(rng, n, u_lo, u_hi, w_lo, w_hi, kind):
    """Uniform-by-area samples on the ribbon/apron strip via rejection on the
    area element (1 + w kappa)/cos(beta)."""
    pts, nrm = [], []
    got = 0
    wmax = max(abs(w_lo), abs(w_hi))
    bound = (1.0 + wmax / RADIUS) / math.cos(BANK_TURN if kind == "ribbon" else 0.0)
    while got < n:
        m = int((n - got) * 1.3) + 64
        u = rng.uniform(u_lo, u_hi, m)
        w = rng.uniform(w_lo, w_hi, m)
        _, _, _, k = centreline(u)
        dens = 1.0 + w * k
        if kind == "ribbon":
            dens = dens / np.cos(bank(u))
        keep = rng.uniform(0.0, bound, m) < dens
        u, w = u[keep], w[keep]
        p, nv = _surface_point(u, w, kind)
        pts.append(p)
        nrm.append(nv)
        got += len(u)
    return np.concatenate(pts)[:n], np.concatenate(nrm)[:n]


def _sample_wall(rng, n, u_lo, u_hi, w, z_lo_fn, height):
    pts, nrm = [], []
    got = 0
    bound = 1.0 + abs(w) / RADIUS
    while got < n:
        m = int((n - got) * 1.3) + 64
        u = rng.uniform(u_lo, u_hi, m)
        x, y, h, k, out = _frame(u)
        keep = rng.uniform(0.0, bound, m) < (1.0 + w * k)
        u, x, y, out = u[keep], x[keep], y[keep], out[keep]
        z0 = z_lo_fn(u)
        t = rng.uniform(0.0, height, len(u))
        p = np.stack([x + w * out[:, 0], y + w * out[:, 1], z0 + t], -1)
        nv = np.stack([-out[:, 0], -out[:, 1], np.zeros(len(u))], -1)
        pts.append(p)
        nrm.append(nv)
        got += len(u)
    return np.concatenate(pts)[:n], np.concatenate(nrm)[:n]


@functools.lru_cache(maxsize=4)
def post_positions(seed: int = 0):
    """Fence posts every 10 m +- U(-2, 2) m along the outer wall (breaks the
    along-track degeneracy, SURVEY.md §8(c) degeneracy caveat)."""
    rng = np.random.default_rng(np.random.SeedSequence([seed, 7777]))
    base = np.arange(0.0, TRACK_LEN - 1e-9, POST_SPACING)
    u = np.mod(base + rng.uniform(-POST_JITTER, POST_JITTER, len(base)), TRACK_LEN)
    return np.sort(u)


def _sample_posts(rng, n, post_u):
    if n == 0 or len(post_u) == 0:
        return np.zeros((0, 3)), np.zeros((0, 3))
    which = rng.integers(0, len(post_u), n)
    u = post_u[which]
    x, y, h, k, out = _frame(u)
    w_c = HALF_WIDTH + 0.3 + POST_R
    cx = x + w_c * out[:, 0]
    cy = y + w_c * out[:, 1]
    z0 = 2 * HALF_WIDTH * np.tan(bank(u))
    ang = rng.uniform(0.0, 2 * math.pi, n)
    t = rng.uniform(0.0, POST_H, n)
    p = np.stack([cx + POST_R * np.cos(ang), cy + POST_R * np.sin(ang), z0 + t], -1)
    nv = np.stack([np.cos(ang), np.sin(ang), np.zeros(n)], -1)
    return p, nv


BOX_SPACING = 30.0


@functools.lru_cache(maxsize=4)
def box_specs(seed: int = 0):
    """Infield marker boxes every 30 m +- U(-8, 8) m beyond the inner wall (seeded):
    arc position u, lateral offset w, size (a, b, h), yaw. They give scan-to-scan
    registration a second family of vertical structure ('add a
    few seeded infield boxes')."""
    rng = np.random.default_rng(np.random.SeedSequence([seed, 8888]))
    base = np.arange(0.0, TRACK_LEN - 1e-9, BOX_SPACING)
    u = np.mod(base + rng.uniform(-8.0, 8.0, len(base)), TRACK_LEN)
    w = -HALF_WIDTH - APRON - rng.uniform(2.0, 6.0, len(base))
    size = np.stack([rng.uniform(1.5, 4.0, len(base)), rng.uniform(0.8, 2.0, len(base)),
                     rng.uniform(0.8, 2.5, len(base))], -1)
    yaw = rng.uniform(0, np.pi, len(base))
    order = np.argsort(u)
    return u[order], w[order], size[order], yaw[order]


def _box_area(size):
    a, b, h = size[..., 0], size[..., 1], size[..., 2]
    return a * b + 2 * (a + b) * h  # top + 4 sides


def _sample_boxes(rng, n, sel):
    u, w, size, yaw = sel
    if n == 0 or len(u) == 0:
        return np.zeros((0, 3)), np.zeros((0, 3))
    area = _box_area(size)
    which = rng.choice(len(u), n, p=area / area.sum())
    x, y, h, k, out = _frame(u[which])
    cx = x + w[which] * out[:, 0]
    cy = y + w[which] * out[:, 1]
    a, b, hh = size[which, 0], size[which, 1], size[which, 2]
    # face choice by area: 0 top, 1/2 +-a faces (b x h), 3/4 +-b faces (a x h)
    fa = np.stack([a * b, b * hh, b * hh, a * hh, a * hh], -1)
    cum = np.cumsum(fa, 1) / fa.sum(1, keepdims=True)
    r = rng.uniform(size=n)
    face = (r[:, None] > cum).sum(1)
    s1 = rng.uniform(-0.5, 0.5, n)
    s2 = rng.uniform(0.0, 1.0, n)
    lx = np.where(face == 0, s1 * a, np.where(face == 1, 0.5 * a, np.where(face == 2, -0.5 * a, s1 * a)))
    ly = np.where(face == 0, rng.uniform(-0.5, 0.5, n) * b,
                  np.where(face <= 2, s1 * b, np.where(face == 3, 0.5 * b, -0.5 * b)))
    lz = np.where(face == 0, hh, s2 * hh)
    nl = np.stack([np.where(face == 1, 1.0, np.where(face == 2, -1.0, 0.0)),
                   np.where(face == 3, 1.0, np.where(face == 4, -1.0, 0.0)),
                   np.where(face == 0, 1.0, 0.0)], -1)
    cyaw, syaw = np.cos(yaw[which]), np.sin(yaw[which])
    px = cx + cyaw * lx - syaw * ly
    py = cy + syaw * lx + cyaw * ly
    nx = cyaw * nl[:, 0] - syaw * nl[:, 1]
    ny = syaw * nl[:, 0] + cyaw * nl[:, 1]
    return np.stack([px, py, lz], -1), np.stack([nx, ny, nl[:, 2]], -1)


def _areas(u_lo=0.0, u_hi=TRACK_LEN, n_posts=None, box_sel=None):
    """Surface areas (m^2) of the four surface kinds over an arc-length window,
    by midpoint integration of the area elements."""
    uu = np.linspace(u_lo, u_hi, 20001)
    um = 0.5 * (uu[1:] + uu[:-1])
    du = np.diff(uu)
    _, _, _, k = centreline(um)
    beta = bank(um)
    # ribbon: w in [-9, 9]; integral of (1 + w k) dw = 18 (odd term cancels)
    ribbon = np.sum(du * 2 * HALF_WIDTH / np.cos(beta))
    # apron: w in [-15, -9]
    w0, w1 = -HALF_WIDTH - APRON, -HALF_WIDTH
    apron = np.sum(du * ((w1 - w0) + 0.5 * k * (w1 ** 2 - w0 ** 2)))
    outer = np.sum(du * (1 + HALF_WIDTH * k)) * OUTER_WALL_H
    inner = np.sum(du * (1 + (-HALF_WIDTH - APRON) * k)) * INNER_WALL_H
    posts = (n_posts if n_posts is not None else len(post_positions())) * 2 * math.pi * POST_R * POST_H
    boxes = float(_box_area((box_sel if box_sel is not None else box_specs())[2]).sum())
    return np.array([ribbon, apron, outer, inner, posts, boxes])


def _sample_surfaces(rng, n, u_lo, u_hi, post_u):
    """n points uniform by area on all track surfaces with u in [u_lo, u_hi)."""
    sel_posts = post_u[(post_u >= u_lo) & (post_u < u_hi)] if u_hi - u_lo < TRACK_LEN else post_u
    bu, bw, bs, by = box_specs()
    bm = (bu >= u_lo) & (bu < u_hi) if u_hi - u_lo < TRACK_LEN else np.ones(len(bu), bool)
    box_sel = (bu[bm], bw[bm], bs[bm], by[bm])
    areas = _areas(u_lo, u_hi, len(sel_posts), box_sel)
    counts = rng.multinomial(n, areas / areas.sum())
    parts = []
    p, nv = _sample_strip(rng, counts[0], u_lo, u_hi, -HALF_WIDTH, HALF_WIDTH, "ribbon")
    parts.append((p, nv))
    p, nv = _sample_strip(rng, counts[1], u_lo, u_hi, -HALF_WIDTH - APRON, -HALF_WIDTH, "apron")
    parts.append((p, nv))
    p, nv = _sample_wall(rng, counts[2], u_lo, u_hi, HALF_WIDTH,
                         lambda u: 2 * HALF_WIDTH * np.tan(bank(u)), OUTER_WALL_H)
    parts.append((p, nv))
    p, nv = _sample_wall(rng, counts[3], u_lo, u_hi, -HALF_WIDTH - APRON,
                         lambda u: np.zeros_like(u), INNER_WALL_H)
    parts.append((p, nv))
    p, nv = _sample_posts(rng, counts[4], sel_posts)
    parts.append((p, nv))
    p, nv = _sample_boxes(rng, counts[5], box_sel)
    parts.append((p, nv))
    pts = np.concatenate([a for a, _ in parts])
    nrm = np.concatenate([b for _, b in parts])
    return pts, nrm


@functools.lru_cache(maxsize=4)
def racetrack_map(n: int = 2_000_000, seed: int = 1, sigma: float = NOISE_SIGMA) -> np.ndarray:
    """The C3 map: n points uniform by area over the whole oval (~64k m^2, ~31
    pts/m^2 at 2M), Gaussian noise sigma along the surface normal, shuffled
    (arbitrary storage order). Returns float32 [n, 3], C-contiguous, read-only."""
    rng = np.random.default_rng(np.random.SeedSequence([seed, 1]))
    pts, nrm = _sample_surfaces(rng, n, 0.0, TRACK_LEN, post_positions())
    pts = pts + nrm * rng.normal(0.0, sigma, (len(pts), 1))
    pts = pts[rng.permutation(len(pts))]
    out = np.ascontiguousarray(pts.astype(np.float32))
    out.setflags(write=False)
    return out


def multi_lap_map(n_per_lap: int = 2_000_000, laps: int = 10, seed0: int = 1) -> np.ndarray:
    """C5 map: `laps` independent samples (seeds seed0..), each offset by a per-lap
    drift (N(0, 2 cm) translation, N(0, 0.01 deg) yaw)."""
    parts = []
    for i in range(laps):
        p = racetrack_map(n_per_lap, seed0 + i).astype(np.float64)
        rng = np.random.default_rng(np.random.SeedSequence([seed0 + i, 99]))
        t = rng.normal(0.0, 0.02, 3)
        yaw = math.radians(rng.normal(0.0, 0.01))
        R = euler_to_R(0.0, 0.0, yaw)
        parts.append(p @ R.T + t)
    return np.ascontiguousarray(np.concatenate(parts).astype(np.float32))


# ----------------------------------------------------------------------------
# rigid transforms (input construction only: Euler angles, not the SE(3) exp)
# ----------------------------------------------------------------------------

def euler_to_R(roll: float, pitch: float, yaw: float) -> np.ndarray:
    cr, sr = math.cos(roll), math.sin(roll)
    cp, sp = math.cos(pitch), math.sin(pitch)
    cy, sy = math.cos(yaw), math.sin(yaw)
    Rx = np.array([[1, 0, 0], [0, cr, -sr], [0, sr, cr]])
    Ry = np.array([[cp, 0, sp], [0, 1, 0], [-sp, 0, cp]])
    Rz = np.array([[cy, -sy, 0], [sy, cy, 0], [0, 0, 1]])
    return Rz @ Ry @ Rx


def make_T(R: np.ndarray, t) -> np.ndarray:
    T = np.eye(4)
    T[:3, :3] = R
    T[:3, 3] = t
    return T


def inv_T(T: np.ndarray) -> np.ndarray:
    R, t = T[:3, :3], T[:3, 3]
    return make_T(R.T, -R.T @ t)


def apply_T(T: np.ndarray, pts: np.ndarray) -> np.ndarray:
    """fp64 rigid transform of points, rounded to fp32 (input construction)."""
    p = pts.astype(np.float64) @ T[:3, :3].T + T[:3, 3]
    return np.ascontiguousarray(p.astype(np.float32))


def perturbation(trans: float, rot_deg: float, seed: int) -> np.ndarray:
    """A rigid offset of exactly `trans` metres along a seeded random direction and
    `rot_deg` degrees about a seeded random axis (Rodrigues on the axis)."""
    rng = np.random.default_rng(np.random.SeedSequence([seed, 4242]))
    d = rng.normal(size=3)
    d /= np.linalg.norm(d)
    a = rng.normal(size=3)
    a /= np.linalg.norm(a)
    th = math.radians(rot_deg)
    K = np.array([[0, -a[2], a[1]], [a[2], 0, -a[0]], [-a[1], a[0], 0]])
    R = np.eye(3) + math.sin(th) * K + (1 - math.cos(th)) * (K @ K)
    return make_T(R, trans * d)


# ----------------------------------------------------------------------------
# scans
# ----------------------------------------------------------------------------
SENSOR_HEIGHT = 1.0
ELEV_MIN = math.radians(-15.0)
ELEV_MAX = math.radians(10.0)
RANGE_MAX = 100.0
RANGE_MIN = 1.0
R_REF = 4.0   # m; acceptance min(1, (R_REF/r)^2) gives LiDAR-like 1/r^2 falloff


def vehicle_pose(u: float, w: float = 0.0) -> np.ndarray:
    """Map<-vehicle pose on the racing line: on the banked surface at lateral
    offset w, heading along the track, rolled with the bank, sensor origin
    SENSOR_HEIGHT above the road."""
    x, y, h, k = centreline(np.array([u]))
    beta = float(bank(np.array([u]))[0])
    h = float(h[0])
    out = np.array([math.sin(h), -math.cos(h)])
    p = np.array([x[0] + w * out[0], y[0] + w * out[1], (w + HALF_WIDTH) * math.tan(beta)])
    # roll about the forward axis so the vehicle's left (infield) side is lower
    R = euler_to_R(-beta, 0.0, h)
    p = p + R @ np.array([0.0, 0.0, SENSOR_HEIGHT])
    return make_T(R, p)


@functools.lru_cache(maxsize=64)
def scan(n: int, u: float, seed: int, sigma: float = NOISE_SIGMA):
    """One merged 3-sensor scan (3 x 120 deg azimuth, elevation -15..+10 deg,
    range <= 100 m, acceptance ~ 1/r^2) of n points, expressed in the vehicle
    frame. Returns (points float32 [n,3] read-only, T_true map<-vehicle fp64)."""
    rng = np.random.default_rng(np.random.SeedSequence([seed, 2]))
    T = vehicle_pose(u)
    Rinv = T[:3, :3].T
    org = T[:3, 3]
    post_u = post_positions()
    acc_pts = []
    got = 0
    dens_batch = 4 * n
    tries = 0
    while got < n:
        tries += 1
        pts, nrm = _sample_surfaces(rng, dens_batch, u - 110.0, u + 110.0, post_u)
        pts = pts + nrm * rng.normal(0.0, sigma, (len(pts), 1))
        v = (pts - org) @ Rinv.T          # vehicle frame
        r = np.linalg.norm(v, axis=1)
        elev = np.arcsin(np.clip(v[:, 2] / np.maximum(r, 1e-9), -1, 1))
        ok = (r <= RANGE_MAX) & (r >= RANGE_MIN) & (elev >= ELEV_MIN) & (elev <= ELEV_MAX)
        p_acc = np.minimum(1.0, (R_REF / np.maximum(r, 1e-9)) ** 2)
        ok &= rng.uniform(size=len(r)) < p_acc
        acc_pts.append(v[ok])
        got += int(ok.sum())
        if tries > 200:
            raise RuntimeError("scan sampler failed to reach the requested count")
    v = np.concatenate(acc_pts)
    v = v[rng.choice(len(v), n, replace=False)]
    out = np.ascontiguousarray(v.astype(np.float32))
    out.setflags(write=False)
    return out, T


# ----------------------------------------------------------------------------
# C1: tiny corner scene (ground + two perpendicular walls)
# ----------------------------------------------------------------------------

def corner_scene(seed: int, sigma: float = 0.0) -> np.ndarray:
    """Ground 10x10 m at z=0 (600 pts) + walls x=5 and y=5 (10x2 m, 200 pts each),
    float32 [1000, 3]. The L corner keeps every direction constrained
    (SURVEY.md §8(c) degeneracy caveat)."""
    rng = np.random.default_rng(np.random.SeedSequence([seed, 3]))
    g = np.stack([rng.uniform(-5, 5, 600), rng.uniform(-5, 5, 600), np.zeros(600)], -1)
    g[:, 2] += rng.normal(0, sigma, 600) if sigma > 0 else 0.0
    wx = np.stack([np.full(200, 5.0), rng.uniform(-5, 5, 200), rng.uniform(0, 2, 200)], -1)
    wy = np.stack([rng.uniform(-5, 5, 200), np.full(200, 5.0), rng.uniform(0, 2, 200)], -1)
    if sigma > 0:
        wx[:, 0] += rng.normal(0, sigma, 200)
        wy[:, 1] += rng.normal(0, sigma, 200)
    return np.ascontiguousarray(np.concatenate([g, wx, wy]).astype(np.float32))


C1_T_TRUE = make_T(euler_to_R(math.radians(0.5), math.radians(-0.5), math.radians(3.0)),
                   [0.20, -0.15, 0.05])


def config_c1(exact_copy: bool = False, sigma: float = 0.0):
    """C1: target = corner(seed 11); source = T_true^-1 * (corner(seed 12) or the
    target itself for the exact-copy variant). Returns (src, tgt, T_true, T0)."""
    tgt = corner_scene(11, sigma)
    sample = tgt if exact_copy else corner_scene(12, sigma)
    src = apply_T(inv_T(C1_T_TRUE), sample)
    return src, tgt, C1_T_TRUE.copy(), np.eye(4)


# ----------------------------------------------------------------------------
# configs (BASELINE.json "configs"; the SURVEY §8(d) recipe)
# ----------------------------------------------------------------------------
C2_U0 = 380.0          # straight -> turn transition (bank ramps 9 -> 20 deg)
C2_DU = 6.9            # 69.11 m/s x 0.1 s
C3_U = 380.0


def config_c2(n: int = 30_000):
    """C2 scan-to-scan: target = scan at u0, source = scan at u0 + 6.9 m.
    Returns (src, tgt, T_rel, T0) with T_rel mapping source to target frame."""
    tgt, Tv0 = scan(n, C2_U0, 500)
    src, Tv1 = scan(n, C2_U0 + C2_DU, 501)
    T_rel = inv_T(Tv0) @ Tv1
    T0 = T_rel @ perturbation(0.3, 1.0, 502)
    return src, tgt, T_rel, T0


def config_c3(n_map: int = 2_000_000, n_scan: int = 100_000, scan_seed: int = 1000, u: float = C3_U):
    """C3 scan-to-map: map (seed 1) + one scan (seed scan_seed) at arc length u.
    Returns (scan, map, T_true, T0)."""
    mp = racetrack_map(n_map, 1)
    sc, T = scan(n_scan, u, scan_seed)
    T0 = T @ perturbation(0.5, 1.0, scan_seed + 7)
    return sc, mp, T, T0


def config_c4_scan(i: int, n_scan: int = 100_000):
    """C4 scan i of 256 (seed 1000+i) at u_i = i L / 256 with its own perturbed T0."""
    u = i * TRACK_LEN / 256.0
    sc, T = scan(n_scan, u, 1000 + i)
    return sc, T, T @ perturbation(0.5, 1.0, 1000 + i + 7)


def config_c5(n_per_lap: int = 2_000_000, laps: int = 10, n_scan: int = 100_000, n_scans: int = 10):
    """C5 stress: multi-lap map (laps x n_per_lap points) and a query batch of
    n_scans scans (seeds 2000..) at arc lengths spread over the track, each moved
    into the map frame by its T_true. Returns (map, queries) float32."""
    mp = multi_lap_map(n_per_lap, laps, 1)
    qs = []
    for i in range(n_scans):
        sc, T = scan(n_scan, (i + 0.5) * TRACK_LEN / n_scans, 2000 + i)
        qs.append(apply_T(T, sc))
    return mp, np.ascontiguousarray(np.concatenate(qs).astype(np.float32))


def lattice(side: int = 5) -> np.ndarray:
    """Integer lattice {0..side-1}^3 with idx = (x*side + y)*side + z (the kNN tie
    worked example of SURVEY.md §8(c) "What pins each part")."""
    g = np.arange(side, dtype=np.float32)
    x, y, z = np.meshgrid(g, g, g, indexing="ij")
    return np.ascontiguousarray(np.stack([x.ravel(), y.ravel(), z.ravel()], -1))


def quantised_cloud(n: int, seed: int, half: float = 40.0, step: float = 0.125) -> np.ndarray:
    """Random points on a 1/8 m lattice in [-half, half]^3: every fp32 d2 is exact,
    and exact ties are frequent (exercises the (d2, idx) rule)."""
    rng = np.random.default_rng(np.random.SeedSequence([seed, 5]))
    k = int(half / step)
    return np.ascontiguousarray((rng.integers(-k, k + 1, (n, 3)) * step).astype(np.float32))


def uniform_cloud(n: int, seed: int, lo: float = -10.0, hi: float = 10.0, offset=(0.0, 0.0, 0.0)) -> np.ndarray:
    rng = np.random.default_rng(np.random.SeedSequence([seed, 6]))
    p = rng.uniform(lo, hi, (n, 3)) + np.asarray(offset)
    return np.ascontiguousarray(p.astype(np.float32))


def random_covariances(n: int, seed: int, lo: float = 1e-3, hi: float = 1.0) -> np.ndarray:
    """Generic SPD 3x3 inputs (xx, xy, xz, yy, yz, zz) fp32 [n, 6]: Q diag(l) Q^T with
    Q a uniform random rotation (unit quaternion) and l log-uniform in [lo, hi].
    Input synthesis only (the covariance estimator is not involved)."""
    rng = np.random.default_rng(np.random.SeedSequence([seed, 8]))
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    w, x, y, z = q.T
    Q = np.stack([
        np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)], -1),
        np.stack([2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)], -1),
        np.stack([2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)], -1)], -2)
    lam = np.exp(rng.uniform(np.log(lo), np.log(hi), (n, 3)))
    C = np.einsum("nij,nj,nkj->nik", Q, lam, Q)
    out = np.stack([C[:, 0, 0], C[:, 0, 1], C[:, 0, 2], C[:, 1, 1], C[:, 1, 2], C[:, 2, 2]], -1)
    return np.ascontiguousarray(out.astype(np.float32))
