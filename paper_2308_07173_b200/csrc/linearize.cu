// linearize.cu -- gicp_linearize: gated 1-NN correspondence, Mahalanobis residual,
// Jacobian and the deterministic fp64 reduction of H (21), b (6), e, count.
//
// Paper: d_i = q_i - T p_i (eq_trans_err), cost
// sum d_i^T (C^q_i + R C^p_i R^T)^-1 d_i (eq_trans_err_dist / eq_trans_likelihood,
// l.388-402, readings R1-R4, R12). Per source point (one thread each,
// PPT points per thread, fixed mapping):
//   p' = R p + t in fp64 (FMA chain of the header), s = fl32(p')
//   j* = argmin over ALL targets of (d2(s, q_j), j): voxel-grid search with the
//        conservative stop rule of knn.cu, pruned at the gate r
//   inlier iff d2 < fl32(r*r); d = q - p' (fp64 -> fp32);
//   A = C^q + R C^p R^T, M = A^-1 (fp32 adjugate), J = [skew(p') | -I]
//   H += J^T M J, b += J^T M d, e += d^T M d  (fp64 accumulators)
// Reduction: per-thread fp64 sums -> warp shuffle tree -> block tree -> block
// partials [nblocks][29] -> the last block to finish sums them in block order.
// Every step has a fixed order, so out29 is bitwise reproducible and independent
// of the SM count / scheduling.
#include <cstdio>
#include <cstdlib>

#include "gicp_internal.cuh"
#include "lin_device.cuh"

namespace gicp {
namespace {

constexpr int kLinBlock = 256;
constexpr int kPPT = 1;                       // points per team
constexpr int kTeam = GICP_LIN_TEAM;          // lanes per point (adjacent lanes of a warp)
constexpr int kPPB = kLinBlock / kTeam * kPPT;  // points per block (fixed: defines the partition)
static_assert(kPPB == kLinPPB, "kLinPPB (gicp_internal.cuh) is the partition");
constexpr int kNumAcc = 28;                   // H(21) b(6) e(1); count kept separately
constexpr int kNV = 31;                       // reduced values: 28 + count + (DUAL) e_old + count_old
constexpr int kMaxRing = 16;
#ifndef GICP_LIN_PROF
#define GICP_LIN_PROF 0  // diagnostics build: search stage counts and warp-duration histogram
#endif
#if GICP_LIN_PROF
__device__ unsigned long long g_lprof[80];  // [0..3] stage counts, [4] max search cycles, [5] sum search, [6] sum total,
                                            // [7] max total, [8..39] log2 hist search, [40..71] log2 hist total
#define LPROF(x) x
#else
#define LPROF(x)
#endif
#ifndef GICP_LIN_MINB
#define GICP_LIN_MINB 4  // blocks per SM the fused / terms kernels are compiled for
#endif
#ifndef GICP_LIN_STREAM
#define GICP_LIN_STREAM 0  // 1: per-point streams (source, certificates, correspondences, queue) evict-first
#endif
#if GICP_LIN_STREAM
#define LDS_(p) __ldcs(p)
#define STS_(p, v) __stcs((p), (v))
#else
#define LDS_(p) (*(p))
#define STS_(p, v) (*(p) = (v))
#endif
#ifndef GICP_TERMS_MINB
#define GICP_TERMS_MINB GICP_LIN_MINB  // the terms kernel (split evaluation; 4: 0.809, 5: 0.870, 6: 0.922 ms -- spills)
#endif
#ifndef GICP_TRIAL_MINB
#define GICP_TRIAL_MINB 8  // the trial (error-only) terms kernel: 32 registers (4: 0.132, 6: 0.114, 8: 0.111 ms)
#endif
#ifndef GICP_LIN_WARM
#define GICP_LIN_WARM 0
#endif
#ifndef GICP_LIN_UNROLL
#define GICP_LIN_UNROLL 4
#endif
constexpr int kUnroll = GICP_LIN_UNROLL;  // candidates loaded together in the level-0 scan



struct Levels {
    Grid lv[kMaxLevels];
    int n;
    int ring_level;  // finest level with cell >= r/2: rings there reach the gate in <= 3 steps
    int coarse_ok;   // level 1 may host the lockstep cube stage (Pose::coarse)
    const int2* adj_oc[2];  // level-0 and level-1 voxel adjacency lists (index.cu)
    const int2* adj_rng[2];
};

// Exact gated 1-NN: best = smallest (d2 bits << 32 | original index) over all
// targets whenever that d2 < r2; bp = its coordinates. WARP-SYNCHRONOUS: all 32
// lanes call it (`active` = the lane has a point). Level 0's 27-voxel cube is
// gathered (27 independent probes) and scanned as one flattened stream per lane
// in lockstep (no divergent per-voxel loops); the few points the stop rule (no
// unsearched point below min(best, r2)) does not settle continue per lane:
// coarser levels up to `ring_level`, then ring expansion there.
// the 27 cells of a cube, own cell first, then faces, edges, corners (nearest
// first): code = (dx + 1) + 3 (dy + 1) + 9 (dz + 1)
__constant__ int c_cube27[27] = {13, 12, 14, 10, 16, 4, 22, 9, 11, 15, 17, 3, 5, 21, 23, 1, 7, 19, 25, 0, 2, 6, 8, 18, 20, 24, 26};

// LEAN (k_lin_search's first pass): only the level-0 cube through adjacency lists;
// a lane whose own voxel has no list, or whose cube does not settle the search,
// returns overflow = 2 untouched otherwise and is searched again in full (the
// result is the same exact minimum: the full search repeats the same stage 1)
template <bool CERT, int UNR = kUnroll, bool LEAN = false>
__device__ __forceinline__ void nn_search(const float4* __restrict__ pts, const Levels& lvs, bool active, float qx,
                                          float qy, float qz, float r2, unsigned long long& best, int& bj,
                                          int& overflow, const int t, float& rho, const int l0,
                                          const unsigned long long warm = kEmptyKey, const int warm_j = -1) {
    // the key (d2 bits << 32 | original index) is kept as two words: the common
    // case (d2 larger) is one 32-bit compare, and only the sorted position of the
    // winner is tracked (its coordinates are loaded once, by the caller)
    // warm start (GICP_LIN_WARM): a real candidate's key (the previous
    // correspondence at the new search point) bounds the search from the start;
    // the minimum over all points is unchanged, the pruning is tighter
    unsigned bh = (unsigned)(warm >> 32), bo = (unsigned)(warm & 0xffffffffu);
    overflow = 0;
    bj = warm_j;
    // certificate of the result for the next iteration (R27): the second-smallest
    // scanned d2 and the smallest lower bound of the voxels left unscanned
    unsigned sh2 = 0xffffffffu;
    float lbp = __int_as_float(0x7f800000);
    rho = -1.0f;
    auto bound = [&]() { return fminf(__uint_as_float(bh), r2); };
    LPROF(int ncand = 0; int nvox = 0;)
    auto consider_p = [&](int j, const float4 p) {
        LPROF(++ncand;)
        const unsigned h = __float_as_uint(dist2(qx, qy, qz, p.x, p.y, p.z));
        const unsigned o = __float_as_uint(p.w);
        // (d2 bits, original index) as one 64-bit compare
        const bool better = (((unsigned long long)h << 32) | o) < (((unsigned long long)bh << 32) | bo);
#if GICP_LIN_WARM
        if (CERT) sh2 = better ? bh : ((h < sh2 && o != bo) ? h : sh2);  // (the warm key scanned again: skip)
#else
        if (CERT) sh2 = better ? bh : min(h, sh2);  // (stage 1 scans every point once)
#endif
        bh = better ? h : bh;
        bo = better ? o : bo;
        bj = better ? j : bj;
    };
    auto consider = [&](int j) { consider_p(j, __ldg(pts + j)); };
    // rho = half the gap between the best distance and every other point's lower
    // bound, minus a rounding margin: a search point that moved less than rho keeps
    // this nearest neighbour (distances change by at most the move)
    // The certificate also keeps the pair inside the gate: rho <= (r - d1) minus the
    // same rounding margin, so a carried pair is an inlier without re-measuring it
    // (k_lin_cert then needs no load of the target point)
    auto certify = [&](float m2) {
        const float l2 = fminf(fminf(__uint_as_float(sh2), lbp * kRel), m2);
        LPROF({
            atomicAdd(&g_lprof[64], 1ull);
            if (l2 == __uint_as_float(sh2)) atomicAdd(&g_lprof[65], 1ull);
            else if (l2 == lbp * kRel) atomicAdd(&g_lprof[66], 1ull);
            else atomicAdd(&g_lprof[67], 1ull);
        })
        const float d1 = sqrtf(__uint_as_float(bh)), dl = sqrtf(l2), r = sqrtf(r2);
        rho = fminf(0.5f * (dl - d1) - 1e-6f * (dl + d1) - 1e-6f, (r - d1) - 1e-6f * (r + d1) - 1e-6f);
    };
    auto finish = [&]() {
        best = ((unsigned long long)bh << 32) | bo;
        LPROF(if (ncand) atomicAdd(&g_lprof[75], (unsigned long long)ncand);)
    };
    // the team's lanes split the level-0 candidates; their bests combine by a
    // butterfly min of the (d2 bits, original index) keys after every voxel
    auto team_min = [&]() {
#pragma unroll
        for (int o = 1; o < kTeam; o <<= 1) {
            const unsigned ph = __shfl_xor_sync(0xffffffffu, bh, o), po = __shfl_xor_sync(0xffffffffu, bo, o);
            const int pj = __shfl_xor_sync(0xffffffffu, bj, o);
            const bool better = ph < bh || (ph == bh && po < bo);
            bh = better ? ph : bh;
            bo = better ? po : bo;
            bj = better ? pj : bj;
        }
    };
    auto scan = [&](int2 rng) {
        for (int j = rng.x; j < rng.y; ++j) consider(j);
    };
    // (1) level 0, the 27-voxel cube, lanes in lockstep
    {
        const Grid& g = lvs.lv[l0];
        const int2* __restrict__ adj_oc = lvs.adj_oc[l0];
        const int2* __restrict__ adj_rng = lvs.adj_rng[l0];
        const QGeom G = make_geom(g, qx, qy, qz);
        const float s = g.cell, slack = g.slack;
        int a0 = 0, a1 = 0;
        bool use_adj = false;
        if (active && adj_oc != nullptr) {
            const int2 own = cell_lookup(g, G.cx, G.cy, G.cz);
            if (own.y > own.x) {
                use_adj = true;
                const int2 oc = __ldg(adj_oc + own.x);
                a0 = oc.x;
                a1 = oc.x + oc.y;
            }
        }
        if (LEAN && active && !use_adj) {  // no adjacency list: the full search
            overflow = 2;
            active = false;
        }
        const float lox = axis_gap(-1, G.fx, s, slack), hix = axis_gap(1, G.fx, s, slack);
        const float loy = axis_gap(-1, G.fy, s, slack), hiy = axis_gap(1, G.fy, s, slack);
        const float loz = axis_gap(-1, G.fz, s, slack), hiz = axis_gap(1, G.fz, s, slack);
        // a lane without an adjacency list (its own voxel is empty, or the index has
        // none) probes the 27 cells in the entry loop itself, entry k = c_cube27[k]
        // (no per-lane arrays: the search stays in registers)
        auto probe = [&](int c, int& cx, int& cy, int& cz, float& lb2) {
            const int code = c_cube27[c];
            const int dx = (code % 3) - 1, dy = ((code / 3) % 3) - 1, dz = (code / 9) - 1;
            cx = G.cx + dx;
            cy = G.cy + dy;
            cz = G.cz + dz;
            const float gx = dx < 0 ? lox : (dx > 0 ? hix : 0.0f);
            const float gy = dy < 0 ? loy : (dy > 0 ? hiy : 0.0f);
            const float gz = dz < 0 ? loz : (dz > 0 ? hiz : 0.0f);
            lb2 = __fmaf_rn(gz, gz, __fmaf_rn(gy, gy, gx * gx));
            return (unsigned)cx < (unsigned)g.nx && (unsigned)cy < (unsigned)g.ny && (unsigned)cz < (unsigned)g.nz;
        };
        // entry-major, warp-uniform: step k tests every lane's k-th voxel against
        // min(best, r2) (predicated: load, decode, bound) and the lanes whose voxel
        // survives scan it together (inner loop = the longest surviving range).
        // Nearest-first order makes almost every voxel after the own one prunable.
        const int cnt = use_adj ? a1 - a0 : (active ? 27 : 0);
        const int kmax = __reduce_max_sync(0xffffffffu, active ? cnt : 0);
        // the next entry is loaded one entry ahead; candidates go kUnroll at a time
        // (independent loads in flight together: the search is latency-bound)
        int2 ne = make_int2(0, 0);
        if (use_adj && cnt > 0 && kmax > 0) ne = __ldg(adj_rng + a0);
        for (int k = 0; k < kmax; ++k) {
            int2 r = make_int2(0, 0);
            if (k < cnt) {
                float lb2;
                bool inside = true;
                int cx = 0, cy = 0, cz = 0;
                if (LEAN || use_adj) {
                    const int2 e = ne;
                    if (k + 1 < cnt) ne = __ldg(adj_rng + a0 + k + 1);
                    r = adj_range(e);
                    lb2 = adj_lb2((unsigned)e.y, lox, hix, loy, hiy, loz, hiz);
                } else {
                    inside = probe(k, cx, cy, cz, lb2);
                }
                if (!inside) {
                    r = make_int2(0, 0);
                } else if (lb2 * kRel > bound()) {
                    r = make_int2(0, 0);
                    if (CERT) lbp = fminf(lbp, lb2);
                } else if (!LEAN && !use_adj) {
                    r = hash_find(g, cell_key(cx, cy, cz));
                    if (r.y <= r.x) r = make_int2(0, 0);
                }
            }
            const int len = r.y - r.x;
            const int lmax = __reduce_max_sync(0xffffffffu, len);
            LPROF(nvox += len > 0;)
            LPROF(if ((threadIdx.x & 31) == 0) atomicAdd(&g_lprof[77], (unsigned long long)lmax);)
            for (int j = 0; j < lmax; j += UNR * kTeam) {
                float4 pv[UNR];
#pragma unroll
                for (int u = 0; u < UNR; ++u) {
                    const int c = j + u * kTeam + t;
                    if (c < len) pv[u] = __ldg(pts + r.x + c);
                }
#pragma unroll
                for (int u = 0; u < UNR; ++u) {
                    const int c = j + u * kTeam + t;
                    if (c < len) consider_p(r.x + c, pv[u]);
                }
            }
            if (kTeam > 1) team_min();
        }
        LPROF({
            const unsigned a = __reduce_add_sync(0xffffffffu, active ? (unsigned)ncand : 0u);
            const unsigned v = __reduce_add_sync(0xffffffffu, active ? (unsigned)nvox : 0u);
            const unsigned na = __reduce_add_sync(0xffffffffu, active ? 1u : 0u);
            if ((threadIdx.x & 31) == 0) {
                atomicAdd(&g_lprof[74], (unsigned long long)a);
                atomicAdd(&g_lprof[76], (unsigned long long)v);
                atomicAdd(&g_lprof[73], (unsigned long long)na);
                atomicAdd(&g_lprof[78], 1ull);
            }
            ncand = 0;
        })
        if (!active) { finish(); return; }
        const float m = cube_margin(G, s, slack, 1);
        if (m > 0.0f && bound() < m * m * kRel) {
            if (CERT && kTeam == 1 && bh != 0xffffffffu) certify(m * m * kRel);
            finish();
            return;
        }
        if (G.cx <= 1 && G.cx >= g.nx - 2 && G.cy <= 1 && G.cy >= g.ny - 2 && G.cz <= 1 && G.cz >= g.nz - 2) {
            if (CERT && kTeam == 1 && bh != 0xffffffffu) certify(__int_as_float(0x7f800000));  // the cube holds the whole grid
            finish();
            return;
        }
    }
    if constexpr (LEAN) {  // the cube did not settle it: the full search
        overflow = 2;
        finish();
        return;
    }
    // (2) per lane: coarser levels' cubes up to ring_level, then rings there
    LPROF(atomicAdd(&g_lprof[1], 1ull);)
    const int ring_level = max(lvs.ring_level, l0);
    for (int l = l0 + 1; l <= ring_level; ++l) {
        const Grid& g = lvs.lv[l];
        const QGeom G = make_geom(g, qx, qy, qz);
        const float s = g.cell, slack = g.slack;
        for (int dz = -1; dz <= 1; ++dz)
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    const float gx = axis_gap(dx, G.fx, s, slack), gy = axis_gap(dy, G.fy, s, slack),
                                gz = axis_gap(dz, G.fz, s, slack);
                    if (__fmaf_rn(gz, gz, __fmaf_rn(gy, gy, gx * gx)) * kRel > bound()) continue;
                    scan(cell_lookup(g, G.cx + dx, G.cy + dy, G.cz + dz));
                }
        const float m = cube_margin(G, s, slack, 1);
        if (m > 0.0f && bound() < m * m * kRel) { finish(); return; }
        if (G.cx <= 1 && G.cx >= g.nx - 2 && G.cy <= 1 && G.cy >= g.ny - 2 && G.cz <= 1 && G.cz >= g.nz - 2) {
            finish();
            return;
        }
    }
    {
        const Grid& g = lvs.lv[ring_level];
        const QGeom G = make_geom(g, qx, qy, qz);
        const float s = g.cell, slack = g.slack;
        const int R0 = max(max(max(-G.cx, G.cx - (g.nx - 1)), max(-G.cy, G.cy - (g.ny - 1))),
                           max(-G.cz, G.cz - (g.nz - 1)));
        LPROF(atomicAdd(&g_lprof[2], 1ull);)
        for (int R = 2;; ++R) {
            if (R < R0) R = R0;
            if (R > max(R0, 1) + kMaxRing) {
                LPROF(atomicAdd(&g_lprof[3], 1ull);)
                overflow = 1;
                { finish(); return; }
            }
            const int z0 = max(-R, -G.cz), z1 = min(R, g.nz - 1 - G.cz);
            const int y0 = max(-R, -G.cy), y1 = min(R, g.ny - 1 - G.cy);
            const int x0 = max(-R, -G.cx), x1 = min(R, g.nx - 1 - G.cx);
            for (int dz = z0; dz <= z1; ++dz) {
                const float gz = axis_gap(dz, G.fz, s, slack);
                for (int dy = y0; dy <= y1; ++dy) {
                    const float gy = axis_gap(dy, G.fy, s, slack);
                    if (__fmaf_rn(gz, gz, gy * gy) * kRel > bound()) continue;
                    auto visit = [&](int dx) {
                        const float gx = axis_gap(dx, G.fx, s, slack);
                        const float lb2 = __fmaf_rn(gz, gz, __fmaf_rn(gy, gy, gx * gx));
                        if (lb2 * kRel > bound()) return;
                        scan(cell_lookup(g, G.cx + dx, G.cy + dy, G.cz + dz));
                    };
                    if (dz == -R || dz == R || dy == -R || dy == R) {
                        for (int dx = x0; dx <= x1; ++dx) visit(dx);
                    } else {
                        if (-R >= x0) visit(-R);
                        if (R <= x1) visit(R);
                    }
                }
            }
            const float mR = cube_margin(G, s, slack, R);
            if (mR > 0.0f && bound() < mR * mR * kRel) { finish(); return; }
            if (G.cx - R <= 0 && G.cx + R >= g.nx - 1 && G.cy - R <= 0 && G.cy + R >= g.ny - 1 && G.cz - R <= 0 &&
                G.cz + R >= g.nz - 1)
                { finish(); return; }
        }
    }
    finish();
}

// brute-force fallback for overflowed searches (the caller handles one point)
__device__ __forceinline__ void nn_bruteforce(const float4* __restrict__ pts, int64_t n, float qx, float qy, float qz,
                                              unsigned long long& best, int& bj) {
    best = kEmptyKey;
    for (int64_t j = 0; j < n; ++j) {
        const float4 p = __ldg(pts + j);
        const float d2 = dist2(qx, qy, qz, p.x, p.y, p.z);
        const unsigned long long key = ((unsigned long long)__float_as_uint(d2) << 32) | __float_as_uint(p.w);
        if (key < best) {
            best = key;
            bj = (int)j;
        }
    }
}

// target covariance of a correspondence: the index's sorted-order copy (2 x
// float4, one 32-B sector, spatially coherent) or the caller's original order
__device__ __forceinline__ void load_cov_sorted(const float4* __restrict__ c8, int spos, float o[6]) {
    const float4 a = __ldg(c8 + 2 * (int64_t)spos), b = __ldg(c8 + 2 * (int64_t)spos + 1);
    o[0] = a.x;
    o[1] = a.y;
    o[2] = a.z;
    o[3] = a.w;
    o[4] = b.x;
    o[5] = b.y;
}

__device__ __forceinline__ void load_cov6_stream(const float* __restrict__ c, int64_t row, float o[6]) {
    const float2* p = reinterpret_cast<const float2*>(c + row * 6);
    const float2 a = LDS_(p), b = LDS_(p + 1), d = LDS_(p + 2);
    o[0] = a.x;
    o[1] = a.y;
    o[2] = b.x;
    o[3] = b.y;
    o[4] = d.x;
    o[5] = d.y;
}

__device__ __forceinline__ void load_cov6(const float* __restrict__ c, int64_t row, float o[6]) {
    const float2* p = reinterpret_cast<const float2*>(c + row * 6);
    const float2 a = __ldg(p), b = __ldg(p + 1), d = __ldg(p + 2);
    o[0] = a.x;
    o[1] = a.y;
    o[2] = b.x;
    o[3] = b.y;
    o[4] = d.x;
    o[5] = d.y;
}


// the terms of one pair as fp32 values (one point per thread: every fp64 sum of the
// reduction starts from these exact values); returns e
template <bool ERROR_ONLY>
__device__ __forceinline__ float point_terms_at(const Pose& P, const double pp[3], float qx, float qy, float qz,
                                                const float cp[6], const float cq[6], float t[27]) {
    const float dx = (float)((double)qx - pp[0]);
    const float dy = (float)((double)qy - pp[1]);
    const float dz = (float)((double)qz - pp[2]);
    return point_terms<ERROR_ONLY>(P, pp, dx, dy, dz, cp, cq, t);
}

// a thread's values (one point): [0, 27) H and b, 27 e, 28 count, 29 e' (DUAL),
// 30 its count; 0.0f + x, as the fp64 accumulators 0.0 + x were (signed zeros)
constexpr int kTV = 32;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
    return v;
}

// the block's reduction and the launch's epilogue (shared by k_linearize and
// k_lin_terms): warp butterfly + block tree into the block's partial row, the last
// block of a registration sums its partials in a fixed order, the last
// registration signals the launch
template <bool ERROR_ONLY, bool DUAL>
__device__ __forceinline__ void lin_block_finish(const float (&tv)[kTV], const int scan, const int blk, const int nblk,
                                                 const int gblk, double* __restrict__ partials,
                                                 unsigned* __restrict__ done, double* __restrict__ out29,
                                                 volatile unsigned* flag, const unsigned seq, const BatchView& bv) {
    // warp tree
    constexpr int NV = DUAL ? kNV : kNumAcc + 1;
    __shared__ double sh[kLinBlock / 32][kNV];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (ERROR_ONLY) {
        const double v = warp_sum((double)tv[27]), n = warp_sum((double)tv[28]);
        if (lane == 0) {
            sh[wid][27] = v;
            sh[wid][kNumAcc] = n;
        }
    } else {
        // butterfly reduce-scatter of the (up to) 32 values: at the stage of offset
        // o a lane keeps the half of its values whose index bit matches its lane bit
        // and adds its partner's copy of them, so after 5 stages lane L holds the
        // warp sum of value L -- 31 exchanges instead of 5 per value (fixed order)
        // (the first stage exchanges the fp32 values and adds them in fp64: the
        // same sums as from fp64 copies, half the registers)
        double val[16];
        {
            const bool up = lane & 16;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const float send = up ? tv[i] : tv[i + 16];
                const float keep = up ? tv[i + 16] : tv[i];
                val[i] = (double)keep + (double)__shfl_xor_sync(0xffffffffu, send, 16);
            }
        }
#pragma unroll
        for (int h = 8; h >= 1; h >>= 1) {
            const bool up = lane & h;
#pragma unroll
            for (int i = 0; i < h; ++i) {
                const double send = up ? val[i] : val[i + h];
                const double keep = up ? val[i + h] : val[i];
                val[i] = keep + __shfl_xor_sync(0xffffffffu, send, h);
            }
        }
        if (lane < NV) sh[wid][lane] = val[0];
    }
    __syncthreads();
    // block tree: thread c sums component c over the 8 warps in order
    if (threadIdx.x < NV) {
        const int c = threadIdx.x;
        double v = 0.0;
        if (!(ERROR_ONLY && c < 27)) {
#pragma unroll
            for (int w = 0; w < kLinBlock / 32; ++w) v += sh[w][c];
        }
        partials[(int64_t)gblk * kNV + c] = v;
    }
    if (bv.elist) return;  // deferred: k_lin_reduce sums the partials after the launch
    // last block (of the registration): fixed-order sum of its block partials
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = (atomicAdd(done + scan, 1u) == (unsigned)nblk - 1u);
    __syncthreads();
    if (!last) return;
    __threadfence();
    partials += (int64_t)(gblk - blk) * kNV;  // the registration's first block
    out29 += (int64_t)scan * bv.out_stride;
    // 29 components x 8 interleaved sub-sequences (block b goes to sub b % 8), the
    // loads of each thread batched 8 at a time (independent, in flight together),
    // summed in a fixed order: deterministic and latency-tolerant
    constexpr int kSub = 8;
    __shared__ double part[kSub][kNV];
    const int nb = nblk;
    if (threadIdx.x < kSub * NV) {
        const int c = threadIdx.x % NV, sub = threadIdx.x / NV;
        double v = 0.0;
        int b = sub;
        for (; b + 7 * kSub < nb; b += 8 * kSub) {
            double t[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) t[u] = __ldcg(partials + (int64_t)(b + u * kSub) * kNV + c);
#pragma unroll
            for (int u = 0; u < 8; ++u) v += t[u];
        }
        for (; b < nb; b += kSub) v += __ldcg(partials + (int64_t)b * kNV + c);
        part[sub][c] = v;
    }
    __syncthreads();
    if (threadIdx.x < NV) {
        const int c = threadIdx.x;
        double v = 0.0;
#pragma unroll
        for (int sub = 0; sub < kSub; ++sub) v += part[sub][c];
        out29[c] = v;
    }
    if (threadIdx.x == 0) done[scan] = 0u;
    if (bv.btab) {  // the last registration to finish signals the launch
        __shared__ bool fin;
        __threadfence_system();  // every lane's out row (possibly host-mapped) before the ticket
        __syncthreads();
        if (threadIdx.x == 0) fin = (atomicAdd(done + bv.n_scans, 1u) == (unsigned)bv.n_active - 1u);
        __syncthreads();
        if (!fin) return;
        if (threadIdx.x == 0) done[bv.n_scans] = 0u;
    }
    if (flag) {  // out29 may be host-mapped: make it visible before the signal
        __threadfence_system();
        __syncthreads();
        if (threadIdx.x == 0) *flag = seq;
    }
}

// SORTED: target covariances from the index's sorted-order copy; SPOS: corr holds
// sorted positions (internal to gicp_align) instead of original indices; DUAL
// (gicp_align's speculative step): in the same pass also the cost e' with the
// PREVIOUS correspondences corr_old at this T (LM's trial evaluation), values 29-30.
// CERT: correspondence certificates (gicp_align, R27): read cache_old (DUAL) and
// write cache_new; the other callers compile the tracking out
template <bool REUSE, bool ERROR_ONLY, bool SORTED, bool SPOS, bool DUAL, bool CERT, bool PRE = false>
__global__ void __launch_bounds__(kLinBlock, GICP_LIN_MINB) k_linearize(const float* __restrict__ src, const float* __restrict__ src_cov,
                                                         int64_t ns, const float4* __restrict__ pts,
                                                         const float4* __restrict__ pts_orig, Levels lvs, int64_t nt,
                                                         const float* __restrict__ tgt_cov,
                                                         const float4* __restrict__ tgt_cov_sorted, Pose P, float r2,
                                                         int32_t* __restrict__ corr, const int32_t* __restrict__ corr_old,
                                                         double* __restrict__ partials, unsigned* __restrict__ done,
                                                         double* __restrict__ out29, volatile unsigned* flag,
                                                         unsigned seq, BatchView bv, float4* __restrict__ cache_new,
                                                         const float4* __restrict__ cache_old) {
    LPROF(const long long tk0 = clock64();)
    // batched launches: this block's registration, its block index within it and
    // its point range; every registration is partitioned exactly like a single
    // launch over its own points, so its result is bitwise the single one
    int scan = 0, blk = blockIdx.x, nblk = gridDim.x;
    int gblk = blockIdx.x;  // the block's slot in the partials (batched: its full-table index)
    int64_t p0 = 0, pend = ns;
    if (bv.btab) {
        const int4 e = bv.btab[blockIdx.x];
        scan = e.x;
        blk = e.y;
        nblk = e.z;
        gblk = e.w;
        if (!bv.poses[bv.ereg ? bv.ereg[scan] : scan].active) return;  // block-uniform: converged registration
        p0 = bv.offs[scan];
        pend = bv.offs[scan + 1];
    }
    __shared__ Pose sP;
    if (threadIdx.x == 0) sP = bv.btab ? bv.poses[bv.ereg ? bv.ereg[scan] : scan] : P;
    __syncthreads();
    // correspondence buffers: single launches use (corr, corr_old) as given; a
    // batched registration reads its current buffer (REUSE / DUAL's old) and
    // writes the other one
    if (bv.btab) {
        int32_t* cur = sP.cur ? const_cast<int32_t*>(corr_old) : corr;
        int32_t* oth = sP.cur ? corr : const_cast<int32_t*>(corr_old);
        corr = (REUSE && !PRE) ? cur : oth;  // PRE: this round's correspondences (k_lin_search)
        corr_old = cur;
        if (CERT) {  // the certificates follow their correspondence buffers
            float4* ccur = sP.cur ? const_cast<float4*>(cache_old) : cache_new;
            float4* coth = sP.cur ? cache_new : const_cast<float4*>(cache_old);
            cache_new = coth;
            cache_old = ccur;
        }
    }
    static_assert(kPPT == 1, "one point per thread: its terms are the fp32 values tv");
    float tv[kTV];
#pragma unroll
    for (int c = 0; c < kTV; ++c) tv[c] = 0.0f;
    const int tl = (int)(threadIdx.x % kTeam);  // lane within the point's team
    const int64_t base = p0 + (int64_t)blk * kPPB + threadIdx.x / kTeam;
#pragma unroll 1
    for (int k = 0; k < kPPT; ++k) {
        const int64_t i = base + (int64_t)k * (kLinBlock / kTeam);
        const bool active = i < pend;  // warp-uniform loop: every lane reaches the search
        double pp[3] = {0.0, 0.0, 0.0};
        if (active) {
            const double px = src[3 * i], py = src[3 * i + 1], pz = src[3 * i + 2];
#pragma unroll
            for (int a = 0; a < 3; ++a)
                pp[a] = __fma_rn(sP.R[3 * a + 2], pz, __fma_rn(sP.R[3 * a + 1], py, __fma_rn(sP.R[3 * a], px, sP.t[a])));
        }
        int orig = -1, spos = -1;
        float qx = 0.f, qy = 0.f, qz = 0.f;
        if (REUSE) {
            if (active) {
                const int c = corr[i];
                if (c >= 0 && c < nt) {
                    const float4 q = SPOS ? __ldg(pts + c) : __ldg(pts_orig + c);
                    qx = q.x;
                    qy = q.y;
                    qz = q.z;
                    orig = SPOS ? __float_as_int(q.w) : c;
                    spos = SPOS ? c : __float_as_int(q.w);
                }
            }
        } else {
            const float sx = (float)pp[0], sy = (float)pp[1], sz = (float)pp[2];
            // certificate check (R27): the previous correspondence stays the nearest
            // neighbour while the search point moved less than its rho
            bool cached = false;
            float4 cc = make_float4(0.f, 0.f, 0.f, -1.f);
            if (DUAL && CERT && cache_old && active) {
                cc = __ldg(cache_old + i);
                if (cc.w > 0.0f) {
                    const double ex = (double)sx - cc.x, ey = (double)sy - cc.y, ez = (double)sz - cc.z;
                    cached = sqrt(ex * ex + ey * ey + ez * ez) < (double)cc.w;
                }
            }
            LPROF(if (active) atomicAdd(&g_lprof[72], cached ? 1ull : 0ull);)
            LPROF(if (active) atomicAdd(&g_lprof[79], 1ull);)
            unsigned long long best;
            int bj, ovf;
            float rho;
            LPROF(const long long t0 = clock64();)
            unsigned long long warm = kEmptyKey;
            int warm_j = -1;
#if GICP_LIN_WARM
            if (DUAL && SPOS && active && !cached) {
                const int c = corr_old[i];
                if (c >= 0 && c < nt) {
                    const float4 q = __ldg(pts + c);
                    warm = ((unsigned long long)__float_as_uint(dist2(sx, sy, sz, q.x, q.y, q.z)) << 32) |
                           __float_as_uint(q.w);
                    warm_j = c;
                }
            }
#endif
            nn_search<CERT>(pts, lvs, active && !cached, sx, sy, sz, r2, best, bj, ovf, tl, rho,
                            (sP.coarse && lvs.coarse_ok) ? 1 : 0, warm, warm_j);
            LPROF({
                const unsigned dt = (unsigned)min(clock64() - t0, 0xffffffffll);
                const unsigned mx = __reduce_max_sync(0xffffffffu, dt);
                if ((threadIdx.x & 31) == 0) {
                    atomicAdd(&g_lprof[0], 1ull);
                    atomicAdd(&g_lprof[5], (unsigned long long)mx);
                    atomicMax(&g_lprof[4], (unsigned long long)mx);
                    atomicAdd(&g_lprof[8 + min(31, 31 - __clz(mx | 1))], 1ull);
                }
            })
            if (active) {
                if (cached) {  // the certified pair: its key at the new search point
                    bj = SPOS ? corr_old[i] : __float_as_int(__ldg(pts_orig + corr_old[i]).w);
                    const float4 q = __ldg(pts + bj);
                    best = ((unsigned long long)__float_as_uint(dist2(sx, sy, sz, q.x, q.y, q.z)) << 32) |
                           __float_as_uint(q.w);
                    ovf = 0;
                    rho = cc.w;
                }
                if (ovf) nn_bruteforce(pts, nt, sx, sy, sz, best, bj);
                const float bd2 = __uint_as_float((unsigned)(best >> 32));
                const bool inl = best != kEmptyKey && bd2 < r2;
                orig = inl ? (int)(best & 0xffffffffu) : -1;
                spos = inl ? bj : -1;
                if (corr && tl == 0) corr[i] = SPOS ? spos : orig;
                if (CERT && cache_new && tl == 0)
                    cache_new[i] = cached ? cc : make_float4(sx, sy, sz, (inl && !ovf) ? rho : -1.0f);
                if (inl) {
                    const float4 q = __ldg(pts + bj);
                    qx = q.x;
                    qy = q.y;
                    qz = q.z;
                }
            }
        }
        if (!active) continue;
        float cp[6], cq[6];
        // lane 0 of the team adds the new pair, the last lane the DUAL trial term
        const bool do_new = tl == 0, do_old = DUAL && tl == kTeam - 1;
        if ((do_new && orig >= 0) || do_old) load_cov6(src_cov, i, cp);
        float e_new = 0.0f;
        if (do_new && orig >= 0) {
            if (SORTED)
                load_cov_sorted(tgt_cov_sorted, spos, cq);
            else
                load_cov6(tgt_cov, orig, cq);
            float t[27];
            e_new = point_terms_at<ERROR_ONLY>(sP, pp, qx, qy, qz, cp, cq, t);
            if (!ERROR_ONLY) {
#pragma unroll
                for (int c = 0; c < 27; ++c) tv[c] = 0.0f + t[c];
            }
            tv[27] = 0.0f + e_new;
            tv[28] = 1.0f;
        }
        if (do_old) {  // the trial cost with the previous correspondences
            const int c = corr_old[i];
            if (c >= 0 && c < nt) {
                if (kTeam == 1 && orig >= 0 && c == (SPOS ? spos : orig)) {
                    tv[29] = 0.0f + e_new;  // the same pair at the same pose: the same term, bitwise
                } else {
                    const float4 q = SPOS ? __ldg(pts + c) : __ldg(pts_orig + c);
                    const int so = SPOS ? c : __float_as_int(q.w);
                    const int oo = SPOS ? __float_as_int(q.w) : c;
                    if (SORTED)
                        load_cov_sorted(tgt_cov_sorted, so, cq);
                    else
                        load_cov6(tgt_cov, oo, cq);
                    float t[27];
                    tv[29] = 0.0f + point_terms_at<true>(sP, pp, q.x, q.y, q.z, cp, cq, t);
                }
                tv[30] = 1.0f;
            }
        }
    }
    LPROF({
        const unsigned dt = (unsigned)min(clock64() - tk0, 0xffffffffll);
        const unsigned mx = __reduce_max_sync(0xffffffffu, dt);
        if ((threadIdx.x & 31) == 0) {
            atomicAdd(&g_lprof[6], (unsigned long long)mx);
            atomicMax(&g_lprof[7], (unsigned long long)mx);
            atomicAdd(&g_lprof[40 + min(31, 31 - __clz(mx | 1))], 1ull);
        }
    })
    lin_block_finish<ERROR_ONLY, DUAL>(tv, scan, blk, nblk, gblk, partials, done, out29, flag, seq, bv);
}

// Terms from given correspondences (gicp_align: the trial evaluation e' alone, and
// PRE: the split evaluation's terms after k_lin_cert / k_lin_search; sorted
// positions, sorted target covariances). The same per-point terms and reductions as
// k_linearize, in the same order (bitwise the same result), but laid out for
// latency: every load a point needs (its correspondence, chosen by the pose's `cur`
// read directly, and that target point and covariance) is issued before the block
// waits for its pose, whose copy into shared memory is spread over the first threads.
template <bool ERROR_ONLY, bool DUAL, bool PRE>
__global__ void __launch_bounds__(kLinBlock, ERROR_ONLY ? GICP_TRIAL_MINB : GICP_TERMS_MINB)
    k_lin_terms(const float* __restrict__ src, const float* __restrict__ src_cov, int64_t ns,
                const float4* __restrict__ pts, int64_t nt, const float4* __restrict__ tgt_cov_sorted, Pose P,
                const int32_t* __restrict__ corr, const int32_t* __restrict__ corr_old, double* __restrict__ partials,
                unsigned* __restrict__ done, double* __restrict__ out29, volatile unsigned* flag, unsigned seq,
                BatchView bv) {
    static_assert(sizeof(Pose) % 8 == 0 && sizeof(Pose) / 8 <= kLinBlock, "pose copy");
    int scan = 0, blk = blockIdx.x, nblk = gridDim.x, gblk = blockIdx.x;
    int64_t p0 = 0, pend = ns;
    const Pose* gp = nullptr;  // (the kernel parameter P is not addressed: it would go to the stack)
    if (bv.btab) {
        const int4 e = bv.btab[blockIdx.x];
        scan = e.x;
        blk = e.y;
        nblk = e.z;
        gblk = e.w;
        gp = bv.poses + (bv.ereg ? bv.ereg[scan] : scan);
        p0 = bv.offs[scan];
        pend = bv.offs[scan + 1];
    }
    __shared__ Pose sP;
    if (gp == nullptr) {
        if (threadIdx.x == 0) sP = P;
    } else if (threadIdx.x < sizeof(Pose) / 8) {
        reinterpret_cast<unsigned long long*>(&sP)[threadIdx.x] =
            __ldg(reinterpret_cast<const unsigned long long*>(gp) + threadIdx.x);
    }
    const int64_t i = p0 + (int64_t)blk * kPPB + threadIdx.x;
    const bool active = i < pend;
    // batched: which buffer is current is the pose's `cur` (read directly: no wait
    // for the shared copy); PRE reads the other buffer (this round's) as new and the
    // current as old, REUSE the current alone. Single launches: corr is the written /
    // reused buffer, corr_old the old one.
    bool new_is_a = true;
    if (bv.btab) {
        const bool cur = __ldg(&gp->cur) != 0;
        new_is_a = PRE ? cur : !cur;
    }
    const int32_t* cbuf = new_is_a ? corr : corr_old;
    const int32_t* obuf = new_is_a ? corr_old : corr;
    int cn = -1, co = -1;
    double px = 0.0, py = 0.0, pz = 0.0;
    float cp[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (active) {
        cn = LDS_(cbuf + i);
        if (DUAL) co = LDS_(obuf + i);
        px = LDS_(src + 3 * i);
        py = LDS_(src + 3 * i + 1);
        pz = LDS_(src + 3 * i + 2);
        load_cov6_stream(src_cov, i, cp);
    }
    const bool vn = cn >= 0 && cn < nt, vo = DUAL && co >= 0 && co < nt;
    const float4 q = __ldg(pts + (vn ? cn : 0));
    float cq[6];
    load_cov_sorted(tgt_cov_sorted, vn ? cn : 0, cq);
    __syncthreads();
    if (bv.btab && !sP.active) return;  // block-uniform: converged registration
    float tv[kTV];
#pragma unroll
    for (int c = 0; c < kTV; ++c) tv[c] = 0.0f;
    if (active) {
        double pp[3];
#pragma unroll
        for (int a = 0; a < 3; ++a)
            pp[a] = __fma_rn(sP.R[3 * a + 2], pz, __fma_rn(sP.R[3 * a + 1], py, __fma_rn(sP.R[3 * a], px, sP.t[a])));
        float e_new = 0.0f;
        if (vn) {
            float t[27];
            e_new = point_terms_at<ERROR_ONLY>(sP, pp, q.x, q.y, q.z, cp, cq, t);
            if (!ERROR_ONLY) {
#pragma unroll
                for (int c = 0; c < 27; ++c) tv[c] = 0.0f + t[c];
            }
            tv[27] = 0.0f + e_new;
            tv[28] = 1.0f;
        }
        if (vo) {  // the trial cost with the previous correspondences
            if (vn && co == cn) {
                tv[29] = 0.0f + e_new;  // the same pair at the same pose: the same term, bitwise
            } else {
                const float4 qo = __ldg(pts + co);
                float cqo[6], t[27];
                load_cov_sorted(tgt_cov_sorted, co, cqo);
                tv[29] = 0.0f + point_terms_at<true>(sP, pp, qo.x, qo.y, qo.z, cp, cqo, t);
            }
            tv[30] = 1.0f;
        }
    }
    lin_block_finish<ERROR_ONLY, DUAL>(tv, scan, blk, nblk, gblk, partials, done, out29, flag, seq, bv);
}

// ---------------------------------------------------------------------------
// Split evaluation (GICP_LIN_SPLIT, the certificate paths of gicp_align and
// gicp_align_batched): the fused kernel leaves most lanes of a searching warp idle
// (64 % of the points keep a certified correspondence, the rest search for ~27
// candidates in lockstep) and holds fp64 accumulators through the latency-bound
// search. Instead: (S1) k_lin_cert checks the certificates and queues the points
// that must search; (S2) k_lin_search runs those searches densely (32 searching
// lanes per warp, a persistent grid at the occupancy the search alone needs);
// (S3) k_linearize<PRE> accumulates the terms from the correspondences S1/S2 wrote.
// Every point's search is the same call on the same inputs, and S3 sums the same
// terms in the same order: the result is bitwise the fused kernel's.
// ---------------------------------------------------------------------------

#ifndef GICP_CERT_PPT
#define GICP_CERT_PPT 4  // (1: 0.840, 2: 0.837, 4: 0.811 ms C4 dual)
#endif
constexpr int kCertPPT = GICP_CERT_PPT;  // points per thread of k_lin_cert
// queue entry: the search point and w = i | coarse << 30 | (write base buffers) << 31
template <bool DUAL>
__global__ void __launch_bounds__(kLinBlock / kCertPPT) k_lin_cert(const float* __restrict__ src, int64_t ns,
                                                        const float4* __restrict__ pts, Pose P, float r2, int coarse_ok,
                                                        int32_t* __restrict__ corr, const int32_t* __restrict__ corr_old,
                                                        BatchView bv, float4* __restrict__ cache_new,
                                                        const float4* __restrict__ cache_old, float4* __restrict__ queue,
                                                        unsigned* __restrict__ qcount) {
    int scan = 0, blk = blockIdx.x;
    int64_t p0 = 0, pend = ns;
    if (bv.btab) {
        const int4 e = bv.btab[blockIdx.x];
        scan = e.x;
        blk = e.y;
        if (!bv.poses[bv.ereg ? bv.ereg[scan] : scan].active) return;
        p0 = bv.offs[scan];
        pend = bv.offs[scan + 1];
    }
    __shared__ Pose sP;
    if (threadIdx.x == 0) sP = bv.btab ? bv.poses[bv.ereg ? bv.ereg[scan] : scan] : P;
    __syncthreads();
    unsigned wbase = 1u;  // single launches write (corr, cache_new)
    if (bv.btab) {
        int32_t* cur = sP.cur ? const_cast<int32_t*>(corr_old) : corr;
        int32_t* oth = sP.cur ? corr : const_cast<int32_t*>(corr_old);
        corr = oth;
        corr_old = cur;
        float4* ccur = sP.cur ? const_cast<float4*>(cache_old) : cache_new;
        float4* coth = sP.cur ? cache_new : const_cast<float4*>(cache_old);
        cache_new = coth;
        cache_old = ccur;
        wbase = sP.cur ? 1u : 0u;
    }
    // kCertPPT points per thread (i, i + threads, ...): every load of all of them is
    // issued before any is used (the kernel streams ~60 B a point, latency-bound)
    constexpr int T = kLinBlock / kCertPPT;
    int64_t ii[kCertPPT];
    bool act[kCertPPT], cached[kCertPPT];
    double px[kCertPPT], py[kCertPPT], pz[kCertPPT];
    float4 cc[kCertPPT];
    int bj[kCertPPT];
    float sx[kCertPPT], sy[kCertPPT], sz[kCertPPT];
#pragma unroll
    for (int u = 0; u < kCertPPT; ++u) {
        ii[u] = p0 + (int64_t)blk * kPPB + threadIdx.x + u * T;
        act[u] = ii[u] < pend;
        cached[u] = false;
        cc[u] = make_float4(0.f, 0.f, 0.f, -1.f);
        bj[u] = 0;
        px[u] = py[u] = pz[u] = 0.0;
        if (act[u]) {
            const int64_t i = ii[u];
            px[u] = LDS_(src + 3 * i);
            py[u] = LDS_(src + 3 * i + 1);
            pz[u] = LDS_(src + 3 * i + 2);
            if (DUAL && cache_old) {
                cc[u] = LDS_(cache_old + i);
                bj[u] = LDS_(corr_old + i);
            }
        }
    }
#pragma unroll
    for (int u = 0; u < kCertPPT; ++u) {
        sx[u] = sy[u] = sz[u] = 0.f;
        if (!act[u]) continue;
        double pp[3];
#pragma unroll
        for (int a = 0; a < 3; ++a)
            pp[a] = __fma_rn(sP.R[3 * a + 2], pz[u], __fma_rn(sP.R[3 * a + 1], py[u], __fma_rn(sP.R[3 * a], px[u], sP.t[a])));
        sx[u] = (float)pp[0];
        sy[u] = (float)pp[1];
        sz[u] = (float)pp[2];
        if (DUAL && cache_old) {
            if (cc[u].w > 0.0f) {
                const double ex = (double)sx[u] - cc[u].x, ey = (double)sy[u] - cc[u].y, ez = (double)sz[u] - cc[u].z;
                cached[u] = sqrt(ex * ex + ey * ey + ez * ez) < (double)cc[u].w;
            }
            if (cached[u]) {  // the certified pair (inside the gate by construction of rho)
                STS_(corr + ii[u], bj[u]);
                STS_(cache_new + ii[u], cc[u]);
            }
        }
    }
    // one queue reservation per block (the counter is a single address: per-warp
    // atomics serialise at the L2); slots follow in (point slot, warp) order
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    constexpr int NW = T / 32;
    __shared__ unsigned wcnt[kCertPPT * NW], bbase;
    unsigned m[kCertPPT];
#pragma unroll
    for (int u = 0; u < kCertPPT; ++u) {
        m[u] = __ballot_sync(0xffffffffu, act[u] && !cached[u]);
        if (lane == 0) wcnt[u * NW + wid] = (unsigned)__popc(m[u]);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned tot = 0;
#pragma unroll
        for (int w = 0; w < kCertPPT * NW; ++w) {
            const unsigned c = wcnt[w];
            wcnt[w] = tot;
            tot += c;
        }
        bbase = tot ? atomicAdd(qcount, tot) : 0u;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kCertPPT; ++u) {
        if (act[u] && !cached[u]) {
            const unsigned base = bbase + wcnt[u * NW + wid];
            const unsigned w = (unsigned)ii[u] | ((sP.coarse && coarse_ok) ? (1u << 30) : 0u) | (wbase << 31);
            STS_(queue + base + __popc(m[u] & ((1u << lane) - 1u)),
                 make_float4(sx[u], sy[u], sz[u], __uint_as_float(w)));
        }
    }
}

#ifndef GICP_SEARCH_MINB
#define GICP_SEARCH_MINB 4  // 64 registers: more warps spill, and measured slower (4: 1.64, 5: 2.04, 8: 2.22 ms)
#endif
#ifndef GICP_SEARCH_MINB_LEAN
#define GICP_SEARCH_MINB_LEAN 5  // the lean pass: 48 registers (4: 0.860, 5: 0.845, 6: 0.870 ms C4 dual)
#endif
#ifndef GICP_SEARCH_UNROLL
#define GICP_SEARCH_UNROLL 4  // with the lean first pass (dual launch): 4: 1.12, 2: 1.15 ms
#endif
constexpr int kSearchBlock = 256;
#ifndef GICP_SEARCH_CLAIM
#define GICP_SEARCH_CLAIM 32  // queue entries a warp claims at a time (128: C4 dual 1.12 -> 1.20 ms)
#endif
#ifndef GICP_FULL_PER_WARP
#define GICP_FULL_PER_WARP 32
#endif
#ifndef GICP_COOP_MAX
#define GICP_COOP_MAX 16384  // queue2 sizes searched a warp per point (larger: per lane)
#endif
constexpr unsigned kCoopMax = GICP_COOP_MAX;
#ifndef GICP_SPLIT_MIN
#define GICP_SPLIT_MIN (1 << 20)
#endif
constexpr int64_t kSplitMinPoints = GICP_SPLIT_MIN;
// LEAN: the first pass over the queue (qcount[0] entries, claimed through
// qcount[1]); points it cannot settle go to queue2 (qcount[2], claimed through
// qcount[3]) for the full search (LEAN = false)
template <bool LEAN>
__global__ void __launch_bounds__(kSearchBlock, LEAN ? GICP_SEARCH_MINB_LEAN : GICP_SEARCH_MINB)
    k_lin_search(const float4* __restrict__ pts, Levels lvs, int64_t nt, float r2, int32_t* __restrict__ corr_a,
                 int32_t* __restrict__ corr_b, float4* __restrict__ cache_a, float4* __restrict__ cache_b,
                 const float4* __restrict__ queue, float4* __restrict__ queue2, unsigned* __restrict__ qcount,
                 unsigned max_coop) {
    // each warp claims 32 entries at a time: dynamic balance, and warps in flight
    // work on neighbouring entries
    const unsigned n = LEAN ? qcount[0] : qcount[2];
    if (!LEAN && n <= max_coop) return;  // a small queue2: k_lin_search_coop takes it
    unsigned* claim = qcount + (LEAN ? 1 : 3);
    const float4* q = LEAN ? queue : queue2;
    const int lane = threadIdx.x & 31;
    // (a claim covers kClaim entries, walked 32 at a time: fewer atomics on the one
    // counter address)
    // The full pass takes kPer entries per warp: its points diverge (per-lane coarse
    // levels and rings), so a warp of 32 would serialise them; its queue is small
    // (~3 % of the searches) and the grid has warps to spare.
    constexpr unsigned kPer = LEAN ? 32u : GICP_FULL_PER_WARP;
    constexpr unsigned kClaim = LEAN ? GICP_SEARCH_CLAIM : kPer;
    unsigned w0 = 0, wend = 0;
    for (;;) {
        if (w0 >= wend) {
            unsigned c = 0;
            if (lane == 0) c = atomicAdd(claim, kClaim);
            c = __shfl_sync(0xffffffffu, c, 0);
            if (c >= n) break;
            w0 = c;
            wend = min(c + kClaim, n);
        }
        const unsigned k = w0 + (lane < (int)kPer ? lane : 0x40000000);
        w0 += kPer;
        const bool active = k < wend;  // warp-uniform loop: every lane reaches the search
        float4 e = make_float4(0.f, 0.f, 0.f, 0.f);
        if (active) e = LDS_(q + k);
        const unsigned w = __float_as_uint(e.w);
        unsigned long long best;
        int bj, ovf;
        float rho;
        nn_search<true, GICP_SEARCH_UNROLL, LEAN>(pts, lvs, active, e.x, e.y, e.z, r2, best, bj, ovf, 0, rho,
                                                  (w >> 30) & 1u);
        if (LEAN) {  // the unsettled: to the full search
            const bool push = active && ovf == 2;
            const unsigned m = __ballot_sync(0xffffffffu, push);
            if (m) {
                const int leader = __ffs(m) - 1;
                unsigned base = 0;
                if (lane == leader) base = atomicAdd(qcount + 2, (unsigned)__popc(m));
                base = __shfl_sync(0xffffffffu, base, leader);
                if (push) queue2[base + __popc(m & ((1u << lane) - 1u))] = e;
            }
            if (push) continue;
        }
        if (active) {
            if (ovf) nn_bruteforce(pts, nt, e.x, e.y, e.z, best, bj);
            const float bd2 = __uint_as_float((unsigned)(best >> 32));
            const bool inl = best != kEmptyKey && bd2 < r2;
            const int64_t i = w & 0x3fffffffu;
            STS_((w >> 31 ? corr_a : corr_b) + i, inl ? bj : -1);
            STS_((w >> 31 ? cache_a : cache_b) + i, make_float4(e.x, e.y, e.z, (inl && !ovf) ? rho : -1.0f));
        }
    }
}

// The full pass for a SMALL queue2 (the common case: ~3 % of a dual launch's
// searches): one point per warp, the 32 lanes probing cells and scanning candidates
// together, so a point's chain of dependent probes (27 cells, then rings of 98+) is
// ~4 rounds deep instead of ~125 (the per-lane pass is latency-bound on that chain).
// Same exact minimum (d2 bits, original index) and the same stop rules as
// nn_search; the certificate is issued at the cube exit only, like nn_search.
__global__ void __launch_bounds__(kSearchBlock)
    k_lin_search_coop(const float4* __restrict__ pts, Levels lvs, int64_t nt, float r2, int32_t* __restrict__ corr_a,
                      int32_t* __restrict__ corr_b, float4* __restrict__ cache_a, float4* __restrict__ cache_b,
                      const float4* __restrict__ queue2, unsigned* __restrict__ qcount, unsigned max_coop) {
    const unsigned n = qcount[2];
    if (n > max_coop) return;  // a large queue: the per-lane pass (k_lin_search<false>) takes it
    const int lane = threadIdx.x & 31;
    for (;;) {
        unsigned k = 0;
        if (lane == 0) k = atomicAdd(qcount + 3, 1u);
        k = __shfl_sync(0xffffffffu, k, 0);
        if (k >= n) break;
        const float4 e = __ldg(queue2 + k);
        const unsigned w = __float_as_uint(e.w);
        const int l0 = (int)((w >> 30) & 1u);
        const float qx = e.x, qy = e.y, qz = e.z;
        unsigned bh = 0xffffffffu, bo = 0xffffffffu, sh2 = 0xffffffffu;
        int bj = -1;
        float lbp = __int_as_float(0x7f800000);
        auto consider = [&](int j) {
            const float4 p = __ldg(pts + j);
            const unsigned h = __float_as_uint(dist2(qx, qy, qz, p.x, p.y, p.z));
            const unsigned o = __float_as_uint(p.w);
            const bool better = h < bh || (h == bh && o < bo);
            sh2 = better ? bh : (h < sh2 ? h : sh2);
            bh = better ? h : bh;
            bo = better ? o : bo;
            bj = better ? j : bj;
        };
        // warp minimum of the best keys (every lane gets it); the bound for pruning
        auto wmin_h = [&]() {
            unsigned h = bh;
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) h = min(h, __shfl_xor_sync(0xffffffffu, h, o));
            return h;
        };
        auto bound = [&]() { return fminf(__uint_as_float(wmin_h()), r2); };
        auto scan = [&](int2 r) {
            for (int j = r.x + lane; j < r.y; j += 32) consider(j);
        };
        // cooperative cube at level l: lane c < 27 probes cell c_cube27[c]; cells then
        // taken in that (nearest-first) order, pruned against the warp's bound
        auto cube = [&](int l, bool track) {
            const Grid& g = lvs.lv[l];
            const QGeom G = make_geom(g, qx, qy, qz);
            const float s = g.cell, slack = g.slack;
            int2 rc = make_int2(0, 0);
            float lbc = 0.0f;
            bool in = false;
            if (lane < 27) {
                const int code = c_cube27[lane];
                const int dx = (code % 3) - 1, dy = ((code / 3) % 3) - 1, dz = (code / 9) - 1;
                const int cx = G.cx + dx, cy = G.cy + dy, cz = G.cz + dz;
                in = (unsigned)cx < (unsigned)g.nx && (unsigned)cy < (unsigned)g.ny && (unsigned)cz < (unsigned)g.nz;
                const float gx = axis_gap(dx, G.fx, s, slack), gy = axis_gap(dy, G.fy, s, slack),
                            gz = axis_gap(dz, G.fz, s, slack);
                lbc = __fmaf_rn(gz, gz, __fmaf_rn(gy, gy, gx * gx));
                if (in && !(lbc * kRel > r2)) rc = hash_find(g, cell_key(cx, cy, cz));
            }
            for (int c = 0; c < 27; ++c) {
                const bool ci = __shfl_sync(0xffffffffu, in, c);
                if (!ci) continue;
                const float lb = __shfl_sync(0xffffffffu, lbc, c);
                if (lb * kRel > bound()) {
                    if (track) lbp = fminf(lbp, lb);
                    continue;
                }
                const int2 r = make_int2(__shfl_sync(0xffffffffu, rc.x, c), __shfl_sync(0xffffffffu, rc.y, c));
                if (r.y > r.x) scan(r);
            }
            return G;
        };
        float rho = -1.0f;
        int ovf = 0;
        bool done = false;
        {
            const Grid& g = lvs.lv[l0];
            const QGeom G = cube(l0, true);
            const float m = cube_margin(G, g.cell, g.slack, 1);
            const unsigned wb = wmin_h();
            const float bnd = fminf(__uint_as_float(wb), r2);
            const bool whole = G.cx <= 1 && G.cx >= g.nx - 2 && G.cy <= 1 && G.cy >= g.ny - 2 && G.cz <= 1 &&
                               G.cz >= g.nz - 2;
            if ((m > 0.0f && bnd < m * m * kRel) || whole) {
                done = true;
                if (wb != 0xffffffffu) {  // certificate: second-smallest scanned, pruned bounds, outside
                    // the second smallest over the warp: the winner's own second, the others' bests
                    unsigned wo = bh == wb ? bo : 0xffffffffu;
#pragma unroll
                    for (int o = 16; o >= 1; o >>= 1) wo = min(wo, __shfl_xor_sync(0xffffffffu, wo, o));
                    unsigned s2 = (bh == wb && bo == wo) ? sh2 : bh;
#pragma unroll
                    for (int o = 16; o >= 1; o >>= 1) s2 = min(s2, __shfl_xor_sync(0xffffffffu, s2, o));
                    const float m2 = whole ? __int_as_float(0x7f800000) : m * m * kRel;
                    const float l2 = fminf(fminf(__uint_as_float(s2), lbp * kRel), m2);
                    const float d1 = sqrtf(__uint_as_float(wb)), dl = sqrtf(l2), rr = sqrtf(r2);
                    rho = fminf(0.5f * (dl - d1) - 1e-6f * (dl + d1) - 1e-6f, (rr - d1) - 1e-6f * (rr + d1) - 1e-6f);
                }
            }
        }
        const int ring_level = max(lvs.ring_level, l0);
        for (int l = l0 + 1; !done && l <= ring_level; ++l) {
            const Grid& g = lvs.lv[l];
            const QGeom G = cube(l, false);
            const float m = cube_margin(G, g.cell, g.slack, 1);
            if ((m > 0.0f && bound() < m * m * kRel) ||
                (G.cx <= 1 && G.cx >= g.nx - 2 && G.cy <= 1 && G.cy >= g.ny - 2 && G.cz <= 1 && G.cz >= g.nz - 2))
                done = true;
        }
        if (!done) {  // rings at ring_level, 32 cells probed at a time
            const Grid& g = lvs.lv[ring_level];
            const QGeom G = make_geom(g, qx, qy, qz);
            const float s = g.cell, slack = g.slack;
            const int R0 = max(max(max(-G.cx, G.cx - (g.nx - 1)), max(-G.cy, G.cy - (g.ny - 1))),
                               max(-G.cz, G.cz - (g.nz - 1)));
            for (int R = max(2, R0);; ++R) {
                if (R > max(R0, 1) + kMaxRing) {
                    ovf = 1;
                    break;
                }
                const int side = 2 * R + 1, cells = side * side * side;
                for (int c0 = 0; c0 < cells; c0 += 32) {
                    const float bnd = bound();
                    const int c = c0 + lane;
                    int2 rc = make_int2(0, 0);
                    if (c < cells) {
                        const int dx = c % side - R, dy = (c / side) % side - R, dz = c / (side * side) - R;
                        if (max(max(abs(dx), abs(dy)), abs(dz)) == R) {
                            const float gx = axis_gap(dx, G.fx, s, slack), gy = axis_gap(dy, G.fy, s, slack),
                                        gz = axis_gap(dz, G.fz, s, slack);
                            const float lb2 = __fmaf_rn(gz, gz, __fmaf_rn(gy, gy, gx * gx));
                            if (!(lb2 * kRel > bnd)) rc = cell_lookup(g, G.cx + dx, G.cy + dy, G.cz + dz);
                        }
                    }
                    unsigned m = __ballot_sync(0xffffffffu, rc.y > rc.x);
                    while (m) {
                        const int src = __ffs(m) - 1;
                        m &= m - 1;
                        const int2 r = make_int2(__shfl_sync(0xffffffffu, rc.x, src), __shfl_sync(0xffffffffu, rc.y, src));
                        scan(r);
                    }
                }
                const float mR = cube_margin(G, s, slack, R);
                if (mR > 0.0f && bound() < mR * mR * kRel) break;
                if (G.cx - R <= 0 && G.cx + R >= g.nx - 1 && G.cy - R <= 0 && G.cy + R >= g.ny - 1 && G.cz - R <= 0 &&
                    G.cz + R >= g.nz - 1)
                    break;
            }
        }
        // the winner: the warp's minimum key and its sorted position
        unsigned long long key = ((unsigned long long)bh << 32) | bo;
        int kj = bj;
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
            const unsigned long long pk = __shfl_xor_sync(0xffffffffu, key, o);
            const int pj = __shfl_xor_sync(0xffffffffu, kj, o);
            if (pk < key) {
                key = pk;
                kj = pj;
            }
        }
        if (lane == 0) {
            unsigned long long best = key;
            int j = kj;
            if (ovf) {
                nn_bruteforce(pts, nt, qx, qy, qz, best, j);
                rho = -1.0f;
            }
            const float bd2 = __uint_as_float((unsigned)(best >> 32));
            const bool inl = best != kEmptyKey && bd2 < r2;
            const int64_t i = w & 0x3fffffffu;
            STS_((w >> 31 ? corr_a : corr_b) + i, inl ? j : -1);
            STS_((w >> 31 ? cache_a : cache_b) + i, make_float4(qx, qy, qz, (inl && !ovf) ? rho : -1.0f));
        }
    }
}

// Deferred reduction of a batched launch (BatchView::elist): CTA e sums entry e's
// block partials -- 8 interleaved sub-sequences, each 8 loads at a time, then the 8
// sub-sums in order: the exact order of lin_block_finish's last block, so the rows
// are bitwise the same -- and the last CTA raises the launch's flag. The kernels
// then skip the per-block fence + ticket (30 % of k_lin_terms' stall samples).
template <int NV>
__global__ void __launch_bounds__(kLinBlock) k_lin_reduce(const int2* __restrict__ elist, const int4* __restrict__ btab,
                                                        const double* __restrict__ partials, double* __restrict__ out,
                                                        int out_stride, unsigned* __restrict__ counter,
                                                        volatile unsigned* flag, unsigned seq) {
    const int4 ent = btab[elist[blockIdx.x].x];
    const int scan = ent.x, nb = ent.z;
    const double* pr = partials + (int64_t)ent.w * kNV;  // the entry's first block (blk 0)
    double* o = out + (int64_t)scan * out_stride;
    constexpr int kSub = 8;
    __shared__ double part[kSub][kNV];
    if (threadIdx.x < kSub * NV) {
        const int c = threadIdx.x % NV, sub = threadIdx.x / NV;
        double v = 0.0;
        int b = sub;
        for (; b + 7 * kSub < nb; b += 8 * kSub) {
            double t[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) t[u] = __ldcg(pr + (int64_t)(b + u * kSub) * kNV + c);
#pragma unroll
            for (int u = 0; u < 8; ++u) v += t[u];
        }
        for (; b < nb; b += kSub) v += __ldcg(pr + (int64_t)b * kNV + c);
        part[sub][c] = v;
    }
    __syncthreads();
    if (threadIdx.x < NV) {
        const int c = threadIdx.x;
        double v = 0.0;
#pragma unroll
        for (int sub = 0; sub < kSub; ++sub) v += part[sub][c];
        o[c] = v;
    }
    if (flag) {  // the last CTA signals (the rows may be host-mapped)
        __shared__ bool fin;
        __threadfence_system();
        __syncthreads();
        if (threadIdx.x == 0) fin = atomicAdd(counter, 1u) == gridDim.x - 1u;
        __syncthreads();
        if (!fin) return;
        if (threadIdx.x == 0) {
            *counter = 0u;
            __threadfence_system();
            *flag = seq;
        }
    }
}

__global__ void k_zero29(double* out29) {
    if (threadIdx.x < 29) out29[threadIdx.x] = 0.0;
}

}  // namespace

Pose make_pose(const double T[16], const double* pivot) {
    Pose P{};
    for (int a = 0; a < 3; ++a) {
        for (int b = 0; b < 3; ++b) {
            P.R[3 * a + b] = T[4 * a + b];
            P.Rf[3 * a + b] = (float)T[4 * a + b];
        }
        P.t[a] = T[4 * a + 3];
        P.c[a] = pivot ? pivot[a] : 0.0;
    }
    P.active = 1;
    P.cur = 0;
    return P;
}

int launch_linearize_core(const float* src, const float* src_cov, int64_t ns, const gicp_index_s* tgt,
                          const float* tgt_cov, const Pose& P, float max_corr_dist, int flags, double* out29,
                          int32_t* corr, cudaStream_t s, const LinScratch& scr, const int32_t* corr_old,
                          const BatchView& bv, int64_t nb) {
    volatile float r2v = max_corr_dist * max_corr_dist;  // fp32 product
    const float r2 = r2v;
    const BatchView& bvq = bv;
    Levels lvs;
    lvs.n = tgt->n_levels;
    for (int l = 0; l < kMaxLevels; ++l) lvs.lv[l] = tgt->lv[l < lvs.n ? l : lvs.n - 1];
    lvs.ring_level = lvs.n - 1;
    for (int l = 0; l < lvs.n; ++l)
        if (2.0f * tgt->lv[l].cell >= max_corr_dist) {
            lvs.ring_level = l;
            break;
        }
    // the cube stage at level 1 (kLinCoarse): its 27 cells certify the gate for
    // far-off search points that level 0's cube cannot settle (the search is exact
    // at either level; the choice only moves the work)
    // (per registration: Pose::coarse, set from kLinCoarse for a single launch)
    lvs.coarse_ok = lvs.n > 1 && (tgt->adj_oc1 != nullptr || tgt->adj_oc == nullptr);
    lvs.adj_oc[0] = tgt->adj_oc;
    lvs.adj_rng[0] = tgt->adj_rng;
    lvs.adj_oc[1] = tgt->adj_oc1;
    lvs.adj_rng[1] = tgt->adj_rng1;
    unsigned* done = scr.done;
    double* partials = scr.partials;
    volatile unsigned* flag = scr.flag;
    const unsigned seq = scr.seq;
    // the counter is reset by the last block of every launch, so a preallocated
    // scratch stays valid across calls on one stream
    const bool reuse = flags & GICP_LIN_REUSE_CORR, eonly = flags & GICP_LIN_ERROR_ONLY;
    const bool sorted = tgt->cov_sorted != nullptr && tgt_cov == tgt->cov_attached;
    const bool spos = (flags & kLinCorrSpos) && sorted;
    const bool dual = (flags & kLinDual) && !reuse && !eonly;
#define GICP_LIN_ARGS                                                                                            \
    src, src_cov, ns, tgt->pts, tgt->pts_orig, lvs, tgt->n, tgt_cov, tgt->cov_sorted, P, r2, corr, corr_old, partials, \
        done, out29, flag, seq, bvq, scr.cache_new, scr.cache_old
#define GICP_TERMS_ARGS                                                                                           \
    src, src_cov, ns, tgt->pts, tgt->n, tgt->cov_sorted, P, corr, corr_old, partials, done, out29, flag, seq, bvq
#define GICP_LIN_GO(R, E, S, SP) k_linearize<R, E, S, SP, false, false><<<(unsigned)nb, kLinBlock, 0, s>>>(GICP_LIN_ARGS)
#define GICP_LIN_DUAL(S, SP) k_linearize<false, false, S, SP, true, false><<<(unsigned)nb, kLinBlock, 0, s>>>(GICP_LIN_ARGS)
    // certificates (gicp_align: sorted source, sorted-position correspondences)
    const bool cert = (scr.cache_new || scr.cache_old) && spos && !reuse && !eonly;
#define GICP_LIN_RE(S, SP)           \
    if (reuse && eonly)              \
        GICP_LIN_GO(true, true, S, SP);   \
    else if (reuse)                  \
        GICP_LIN_GO(true, false, S, SP);  \
    else if (eonly)                  \
        GICP_LIN_GO(false, true, S, SP);  \
    else                             \
        GICP_LIN_GO(false, false, S, SP);
    // split evaluation (S1 certificates, S2 dense searches, S3 terms) for the
    // certificate launches over many points (C4, 9M points a launch: dual 1.97 ->
    // 1.39 ms, full 0.62 -> 0.53 ms); a single 100k-point scan (C3) stays fused: its
    // three extra launches and the memset cost more than the denser search saves
    // (C3 align 1.30 -> 1.56 ms split)
    // GICP_LIN_SPLIT_MIN (points, env, read per launch): the threshold; tests force
    // either path to check that they agree bitwise
    int64_t split_min = kSplitMinPoints;
    if (const char* e = getenv("GICP_LIN_SPLIT_MIN")) split_min = atoll(e);
    // GICP_LIN_COOP_MAX (env): the largest full-search queue searched a warp per point
    unsigned coop_max = kCoopMax;
    if (const char* e = getenv("GICP_LIN_COOP_MAX")) coop_max = (unsigned)atoll(e);
    if (cert && scr.queue && ns >= split_min) {
        int rc = check_cuda(cudaMemsetAsync(scr.qcount, 0, 4 * sizeof(unsigned), s), "memset");
        if (rc) return rc;
        if (dual)
            k_lin_cert<true><<<(unsigned)nb, kLinBlock / kCertPPT, 0, s>>>(src, ns, tgt->pts, P, r2, lvs.coarse_ok ? 1 : 0, corr,
                                                                 corr_old, bvq, scr.cache_new, scr.cache_old,
                                                                 scr.queue, scr.qcount);
        else
            k_lin_cert<false><<<(unsigned)nb, kLinBlock / kCertPPT, 0, s>>>(src, ns, tgt->pts, P, r2, lvs.coarse_ok ? 1 : 0, corr,
                                                                  corr_old, bvq, scr.cache_new, scr.cache_old,
                                                                  scr.queue, scr.qcount);
        static int grid = 0, grid2 = 0;
        if (grid == 0) {
            int dev = 0, sms = 0, per = 0, per2 = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_lin_search<true>, kSearchBlock, 0);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per2, k_lin_search<false>, kSearchBlock, 0);
            grid = std::max(1, sms * std::max(per, 1));
            grid2 = std::max(1, sms * std::max(per2, 1));
        }
        // single launches: (corr, cache_new) are the written pair (w bit 31 = 1)
        int32_t* ca = corr;
        int32_t* cb = const_cast<int32_t*>(corr_old);
        const unsigned g2 = (unsigned)std::min<int64_t>(grid, (ns + kSearchBlock - 1) / kSearchBlock);
        k_lin_search<true><<<std::max(g2, 1u), kSearchBlock, 0, s>>>(tgt->pts, lvs, tgt->n, r2, ca, cb, scr.cache_new,
                                                                     const_cast<float4*>(scr.cache_old), scr.queue,
                                                                     scr.queue2, scr.qcount, 0u);
        // the unsettled points: cooperatively (a warp per point) while few, per lane
        // otherwise (each kernel exits at once when the queue is the other's)
        const unsigned g3 = (unsigned)std::min<int64_t>(grid2, std::max<int64_t>(1, g2));
        k_lin_search<false><<<g3, kSearchBlock, 0, s>>>(tgt->pts, lvs, tgt->n, r2, ca, cb, scr.cache_new,
                                                        const_cast<float4*>(scr.cache_old), scr.queue, scr.queue2,
                                                        scr.qcount, coop_max);
        k_lin_search_coop<<<g3, kSearchBlock, 0, s>>>(tgt->pts, lvs, tgt->n, r2, ca, cb, scr.cache_new,
                                                      const_cast<float4*>(scr.cache_old), scr.queue2, scr.qcount,
                                                      coop_max);
        static const bool dbg = getenv("GICP_DEBUG_SPLIT") != nullptr;  // diagnostics: queue sizes
        if (dbg) {
            unsigned q[4];
            cudaMemcpyAsync(q, scr.qcount, sizeof(q), cudaMemcpyDeviceToHost, s);
            cudaStreamSynchronize(s);
            fprintf(stderr, "[gicp split] points %lld queue %u full-search %u\n", (long long)ns, q[0], q[2]);
        }
        if (dual)
            k_lin_terms<false, true, true><<<(unsigned)nb, kLinBlock, 0, s>>>(GICP_TERMS_ARGS);
        else
            k_lin_terms<false, false, true><<<(unsigned)nb, kLinBlock, 0, s>>>(GICP_TERMS_ARGS);
    } else if (cert && dual) {
        k_linearize<false, false, true, true, true, true><<<(unsigned)nb, kLinBlock, 0, s>>>(GICP_LIN_ARGS);
    } else if (cert) {
        k_linearize<false, false, true, true, false, true><<<(unsigned)nb, kLinBlock, 0, s>>>(GICP_LIN_ARGS);
    } else if (dual) {
        if (spos)
            GICP_LIN_DUAL(true, true);
        else if (sorted)
            GICP_LIN_DUAL(true, false);
        else
            GICP_LIN_DUAL(false, false);
    } else if (spos && reuse) {  // given correspondences (the trial evaluation)
        if (eonly)
            k_lin_terms<true, false, false><<<(unsigned)nb, kLinBlock, 0, s>>>(GICP_TERMS_ARGS);
        else
            k_lin_terms<false, false, false><<<(unsigned)nb, kLinBlock, 0, s>>>(GICP_TERMS_ARGS);
    } else if (spos) {
        GICP_LIN_RE(true, true)
    } else if (sorted) {
        GICP_LIN_RE(true, false)
    } else {
        GICP_LIN_RE(false, false)
    }
    if (bv.elist && bv.n_e > 0) {  // the deferred reduction of this launch's entries
        const int rc = check_cuda(cudaGetLastError(), "linearize launch");
        if (rc) return rc;
        if (dual)
            k_lin_reduce<kNV><<<(unsigned)bv.n_e, kLinBlock, 0, s>>>(bv.elist, bv.btab_full, partials, out29,
                                                                    bv.out_stride, done + bv.n_scans, flag, seq);
        else
            k_lin_reduce<kNumAcc + 1><<<(unsigned)bv.n_e, kLinBlock, 0, s>>>(bv.elist, bv.btab_full, partials, out29,
                                                                            bv.out_stride, done + bv.n_scans, flag,
                                                                            seq);
    }
#undef GICP_LIN_DUAL
#undef GICP_LIN_RE
#undef GICP_LIN_GO
#undef GICP_LIN_ARGS
#undef GICP_TERMS_ARGS
    return check_cuda(cudaGetLastError(), "linearize launch");
}

int launch_linearize(const float* src, const float* src_cov, int64_t ns, const gicp_index_s* tgt,
                     const float* tgt_cov, const double T[16], const double* pivot, float max_corr_dist, int flags,
                     double* out29, int32_t* corr, cudaStream_t s, const LinScratch* pre,
                     const int32_t* corr_old) {
    if (ns == 0) {
        k_zero29<<<1, 32, 0, s>>>(out29);
        return check_cuda(cudaGetLastError(), "linearize launch");
    }
    Pose P = make_pose(T, pivot);
    P.coarse = (flags & kLinCoarse) ? 1 : 0;
    const int64_t nb = (ns + kPPB - 1) / kPPB;
    void* scratch = nullptr;
    LinScratch scr;
    if (pre) {
        scr = *pre;
    } else {
        const size_t bytes = linearize_scratch_bytes(ns);
        if (cudaMallocAsync(&scratch, bytes, s) != cudaSuccess) {
            cudaGetLastError();
            return set_error(GICP_ENOMEM, "linearize scratch allocation failed");
        }
        scr.done = (unsigned*)scratch;
        scr.partials = (double*)((char*)scratch + 256);
        int rc = check_cuda(cudaMemsetAsync(scr.done, 0, sizeof(unsigned), s), "memset");
        if (rc) {
            cudaFreeAsync(scratch, s);
            return rc;
        }
    }
    // the counter is reset by the last block of every launch, so a preallocated
    // scratch stays valid across calls on one stream
    if (corr_old) flags |= kLinDual;
    const int rc = launch_linearize_core(src, src_cov, ns, tgt, tgt_cov, P, max_corr_dist, flags, out29, corr, s, scr,
                                         corr_old, BatchView{}, nb);
    if (scratch) cudaFreeAsync(scratch, s);
    return rc;
}

size_t linearize_partials_bytes(int64_t nblocks) { return (size_t)nblocks * kNV * sizeof(double); }

size_t linearize_scratch_bytes(int64_t ns) {
    const int64_t nb = (ns + kPPB - 1) / kPPB;
    return (size_t)nb * kNV * sizeof(double) + 256;
}

}  // namespace gicp

#if GICP_LIN_PROF
// diagnostics builds only (tools/lin_prof.py): read and optionally reset the counters
GICP_API int gicp_debug_lin_prof(unsigned long long* out80, int reset) {
    cudaDeviceSynchronize();
    if (cudaMemcpyFromSymbol(out80, gicp::g_lprof, sizeof(gicp::g_lprof)) != cudaSuccess) return -1;
    if (reset) {
        static const unsigned long long z[80] = {};
        cudaMemcpyToSymbol(gicp::g_lprof, z, sizeof(z));
    }
    return 0;
}
#endif
