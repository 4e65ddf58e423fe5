// knn.cu -- exact kNN on the voxel grid, and the fused kNN + covariance kernel.
//
// Paper: "GPU-based nearest points search and covariance computation" (PAPER.md
// l.413, l.798); the CPU bottleneck it removes is "the corresponding points
// search" during covariance estimation (l.797, l.403-405).
//
// Design:
//  * one thread per query; queries are visited in voxel-sorted order so a warp's
//    32 lanes sit in 1-3 adjacent voxels and read the same candidate lines (L1);
//  * register-resident sorted top-K of 64-bit keys (bits(d2) << 32 | payload);
//    K padded to KCAP (multiple of 4) with 0-keys at the FRONT so the K-th key is
//    always the static slot KCAP-1;
//  * the payload is the candidate's SORTED position (its float4 is then an L1
//    hit for the covariance gather); ties in d2 -- where the definition orders by
//    ORIGINAL index -- are detected on the fly and such queries are recomputed
//    with (d2, original index) keys (EXACT mode);
//  * candidates: the 27 voxels around the query (nearest-first, pruned by box
//    distance), then rings R = 2, 3, ... until no unsearched point can beat the
//    K-th key (conservative geometric stop rule with slack);
//  * queries whose search would exceed kMaxRing rings are queued to a
//    block-per-query brute-force kernel (exact, rare).
#include <cub/cub.cuh>

#include "cov_device.cuh"
#include "gicp_internal.cuh"

namespace gicp {
namespace {

constexpr int kBlock = 128;
constexpr int kMaxRing = 24;
constexpr float kRel = 1.0f - 1.0f / (1 << 20);  // relative safety on squared bounds

// first ring, nearest-first: own voxel, 6 faces, 12 edges, 8 corners
__constant__ signed char c_off27[27][3] = {
    {0, 0, 0},   {-1, 0, 0},  {1, 0, 0},   {0, -1, 0},  {0, 1, 0},   {0, 0, -1},  {0, 0, 1},
    {-1, -1, 0}, {1, -1, 0},  {-1, 1, 0},  {1, 1, 0},   {-1, 0, -1}, {1, 0, -1},  {-1, 0, 1},
    {1, 0, 1},   {0, -1, -1}, {0, 1, -1},  {0, -1, 1},  {0, 1, 1},   {-1, -1, -1}, {1, -1, -1},
    {-1, 1, -1}, {1, 1, -1},  {-1, -1, 1}, {1, -1, 1},  {-1, 1, 1},  {1, 1, 1}};

__device__ __forceinline__ unsigned hi32(unsigned long long k) { return (unsigned)(k >> 32); }

template <int KCAP>
__device__ __forceinline__ void topk_insert(unsigned long long (&L)[KCAP], unsigned long long x) {
    bool below = true;  // caller guarantees x < L[KCAP-1]
#pragma unroll
    for (int r = KCAP - 1; r > 0; --r) {
        const bool gt = x < L[r - 1];
        L[r] = gt ? L[r - 1] : (below ? x : L[r]);
        below = gt;
    }
    L[0] = below ? x : L[0];
}

// compare-and-swap on the d2 bits (high word); ties are handled by the callers
__device__ __forceinline__ void cas_hi(unsigned long long& a, unsigned long long& b) {
    const bool sw = hi32(b) < hi32(a);
    const unsigned long long lo = sw ? b : a;
    b = sw ? a : b;
    a = lo;
}

// Batcher odd-even merge sort network on N register keys. The comparator list is
// generated at compile time (constexpr) so every register index is a constant
// after unrolling. N = 20 -> 103 comparators.
struct SortNet {
    int n;
    unsigned char a[256], b[256];
};

constexpr SortNet make_sortnet(int N) {
    SortNet r{};
    r.n = 0;
    for (int p = 1; p < N; p <<= 1)
        for (int k = p; k >= 1; k >>= 1)
            for (int j = k % p; j + k < N; j += 2 * k)
                for (int i = 0; i < k && i < N - j - k; ++i)
                    if ((i + j) / (2 * p) == (i + j + k) / (2 * p)) {
                        r.a[r.n] = (unsigned char)(i + j);
                        r.b[r.n] = (unsigned char)(i + j + k);
                        ++r.n;
                    }
    return r;
}

template <int N>
__device__ __forceinline__ void sort_network(unsigned long long (&v)[N]) {
    constexpr SortNet net = make_sortnet(N);
#pragma unroll
    for (int c = 0; c < net.n; ++c) cas_hi(v[net.a[c]], v[net.b[c]]);
}

// per-query geometry relative to its own voxel
struct QGeom {
    float qx, qy, qz;
    int cx, cy, cz;
    float fx, fy, fz;  // distance from q to the low faces of its voxel (m)
};

__device__ __forceinline__ QGeom make_geom(const Grid& g, float qx, float qy, float qz) {
    QGeom G;
    G.qx = qx;
    G.qy = qy;
    G.qz = qz;
    G.cx = cell_coord(qx, g.ox, g.inv_cell);
    G.cy = cell_coord(qy, g.oy, g.inv_cell);
    G.cz = cell_coord(qz, g.oz, g.inv_cell);
    const double s = (double)g.cell;
    G.fx = (float)((double)qx - ((double)g.ox + (double)G.cx * s));
    G.fy = (float)((double)qy - ((double)g.oy + (double)G.cy * s));
    G.fz = (float)((double)qz - ((double)g.oz + (double)G.cz * s));
    return G;
}

// lower bound on the distance from q to any point of the voxel at offset d on one axis
__device__ __forceinline__ float axis_gap(int d, float f, float s, float slack) {
    float gap = 0.0f;
    if (d < 0) gap = (float)(-d - 1) * s + f - slack;
    if (d > 0) gap = (float)(d - 1) * s + (s - f) - slack;
    return fmaxf(gap, 0.0f);
}

// the search. EXACT = false: payload = sorted position, tie detection on;
// EXACT = true: payload = original index (the definition's key).
template <int KCAP, bool EXACT>
__device__ __forceinline__ void knn_search(const float4* __restrict__ pts, const HashEntry* __restrict__ H,
                                           const Grid& g, const QGeom& G, unsigned long long (&L)[KCAP], int K,
                                           unsigned& tie_hi, int& overflow) {
#pragma unroll
    for (int r = 0; r < KCAP; ++r) L[r] = (r < KCAP - K) ? 0ull : kEmptyKey;
    tie_hi = 0xffffffffu;
    overflow = 0;
    const float s = g.cell, slack = g.slack;

    auto scan = [&](int2 rng) {
        for (int j = rng.x; j < rng.y; ++j) {
            const float4 p = __ldg(pts + j);
            const float d2 = dist2(G.qx, G.qy, G.qz, p.x, p.y, p.z);
            const unsigned hi = __float_as_uint(d2);
            const unsigned kth = hi32(L[KCAP - 1]);
            if (hi <= kth) {
                const unsigned pay = EXACT ? __float_as_uint(p.w) : (unsigned)j;
                const unsigned long long key = ((unsigned long long)hi << 32) | pay;
                if (!EXACT && hi == kth) tie_hi = min(tie_hi, hi);
                if (key < L[KCAP - 1]) {
                    topk_insert<KCAP>(L, key);
                    if (!EXACT && kth == hi32(L[KCAP - 1])) tie_hi = min(tie_hi, kth);
                }
            }
        }
    };

    const float lo2x = axis_gap(-1, G.fx, s, slack), hi2x = axis_gap(1, G.fx, s, slack);
    const float lo2y = axis_gap(-1, G.fy, s, slack), hi2y = axis_gap(1, G.fy, s, slack);
    const float lo2z = axis_gap(-1, G.fz, s, slack), hi2z = axis_gap(1, G.fz, s, slack);
    // ring 1: 27 voxels nearest-first
    for (int c = 0; c < 27; ++c) {
        const int dx = c_off27[c][0], dy = c_off27[c][1], dz = c_off27[c][2];
        const float gx = dx < 0 ? lo2x : (dx > 0 ? hi2x : 0.0f);
        const float gy = dy < 0 ? lo2y : (dy > 0 ? hi2y : 0.0f);
        const float gz = dz < 0 ? lo2z : (dz > 0 ? hi2z : 0.0f);
        const float lb2 = __fmaf_rn(gz, gz, __fmaf_rn(gy, gy, gx * gx));
        if (lb2 * kRel > __uint_as_float(hi32(L[KCAP - 1]))) continue;  // NaN (not full) -> false
        scan(cell_lookup(H, g, G.cx + dx, G.cy + dy, G.cz + dz));
    }
    // rings R >= 2 until the stop rule holds
    const int R0 = max(max(max(-G.cx, G.cx - (g.nx - 1)), max(-G.cy, G.cy - (g.ny - 1))),
                       max(-G.cz, G.cz - (g.nz - 1)));  // rings below R0 lie outside the grid
    int R = 1;
    while (true) {
        // stop rule after the cube of Chebyshev radius R
        const float mx = fminf(G.fx + R * s, (R + 1) * s - G.fx);
        const float my = fminf(G.fy + R * s, (R + 1) * s - G.fy);
        const float mz = fminf(G.fz + R * s, (R + 1) * s - G.fz);
        const float m = fminf(mx, fminf(my, mz)) - slack;
        const float kth_d2 = __uint_as_float(hi32(L[KCAP - 1]));
        if (m > 0.0f && kth_d2 < m * m * kRel) break;
        const bool covers = G.cx - R <= 0 && G.cx + R >= g.nx - 1 && G.cy - R <= 0 && G.cy + R >= g.ny - 1 &&
                            G.cz - R <= 0 && G.cz + R >= g.nz - 1;
        if (covers) break;  // every voxel searched
        ++R;
        if (R < R0) R = R0;
        if (R > max(R0, 1) + kMaxRing) {
            overflow = 1;
            return;
        }
        const int z0 = max(-R, -G.cz), z1 = min(R, g.nz - 1 - G.cz);
        const int y0 = max(-R, -G.cy), y1 = min(R, g.ny - 1 - G.cy);
        const int x0 = max(-R, -G.cx), x1 = min(R, g.nx - 1 - G.cx);
        for (int dz = z0; dz <= z1; ++dz) {
            const float gz = axis_gap(dz, G.fz, s, slack);
            for (int dy = y0; dy <= y1; ++dy) {
                const float gy = axis_gap(dy, G.fy, s, slack);
                if (__fmaf_rn(gz, gz, gy * gy) * kRel > __uint_as_float(hi32(L[KCAP - 1]))) continue;
                auto visit = [&](int dx) {
                    const float gx = axis_gap(dx, G.fx, s, slack);
                    const float lb2 = __fmaf_rn(gz, gz, __fmaf_rn(gy, gy, gx * gx));
                    if (lb2 * kRel > __uint_as_float(hi32(L[KCAP - 1]))) return;
                    scan(cell_lookup(H, g, G.cx + dx, G.cy + dy, G.cz + dz));
                };
                if (dz == -R || dz == R || dy == -R || dy == R) {
                    for (int dx = x0; dx <= x1; ++dx) visit(dx);
                } else {
                    if (-R >= x0) visit(-R);
                    if (R <= x1) visit(R);
                }
            }
        }
    }
}

// non-EXACT result needs recomputation iff a tie touches the K-th key or two kept
// keys share a d2
template <int KCAP>
__device__ __forceinline__ bool needs_exact(const unsigned long long (&L)[KCAP], int K, unsigned tie_hi) {
    bool fix = (tie_hi == hi32(L[KCAP - 1]));
#pragma unroll
    for (int r = 0; r + 1 < KCAP; ++r)
        if (r >= KCAP - K) fix |= (hi32(L[r]) == hi32(L[r + 1]));
    return fix;
}

// write one row: nbr = original indices, d2; returns nothing. spos_of(r) gives the
// sorted position of slot r.
template <int KCAP, bool EXACT>
__device__ __forceinline__ void write_row(const float4* __restrict__ pts, const float4* __restrict__ pts_orig,
                                          const unsigned long long (&L)[KCAP], int K, int64_t row, int32_t* nbr,
                                          float* d2) {
    if (nbr) {
        int32_t* o = nbr + row * K;
#pragma unroll
        for (int r = 0; r < KCAP; ++r) {
            if (r < KCAP - K) continue;
            const unsigned pay = (unsigned)(L[r] & 0xffffffffu);
            const int orig = EXACT ? (int)pay : __float_as_int(__ldg(pts + pay).w);
            o[r - (KCAP - K)] = orig;
        }
    }
    if (d2) {
        float* o = d2 + row * K;
#pragma unroll
        for (int r = 0; r < KCAP; ++r) {
            if (r < KCAP - K) continue;
            o[r - (KCAP - K)] = __uint_as_float(hi32(L[r]));
        }
    }
}

// covariance of the K kept neighbours (gathered through the sorted float4 array)
template <int KCAP, bool EXACT>
__device__ __forceinline__ void cov_row(const float4* __restrict__ pts, const float4* __restrict__ pts_orig,
                                        const unsigned long long (&L)[KCAP], int K, float eps, float* out6) {
    auto pos = [&](int r) -> int {
        const unsigned pay = (unsigned)(L[r] & 0xffffffffu);
        return EXACT ? __float_as_int(__ldg(pts_orig + pay).w) : (int)pay;
    };
    unsigned long long first = 0ull;
#pragma unroll
    for (int r = 0; r < KCAP; ++r)
        if (r == KCAP - K) first = L[r];
    const float4 p0 = __ldg(pts + (EXACT ? __float_as_int(__ldg(pts_orig + (unsigned)(first & 0xffffffffu)).w)
                                         : (int)(unsigned)(first & 0xffffffffu)));
    float sx = 0.f, sy = 0.f, sz = 0.f;
#pragma unroll
    for (int r = 0; r < KCAP; ++r) {
        if (r < KCAP - K) continue;
        const float4 p = __ldg(pts + pos(r));
        sx += p.x - p0.x;
        sy += p.y - p0.y;
        sz += p.z - p0.z;
    }
    const float invk = 1.0f / (float)K;
    const float mx = sx * invk, my = sy * invk, mz = sz * invk;
    float c00 = 0.f, c01 = 0.f, c02 = 0.f, c11 = 0.f, c12 = 0.f, c22 = 0.f;
#pragma unroll
    for (int r = 0; r < KCAP; ++r) {
        if (r < KCAP - K) continue;
        const float4 p = __ldg(pts + pos(r));
        const float x = (p.x - p0.x) - mx, y = (p.y - p0.y) - my, z = (p.z - p0.z) - mz;
        c00 = fmaf(x, x, c00);
        c01 = fmaf(x, y, c01);
        c02 = fmaf(x, z, c02);
        c11 = fmaf(y, y, c11);
        c12 = fmaf(y, z, c12);
        c22 = fmaf(z, z, c22);
    }
    plane_cov(c00 * invk, c01 * invk, c02 * invk, c11 * invk, c12 * invk, c22 * invk, eps, out6);
}

__device__ __forceinline__ void store_cov(float* cov, int64_t row, const float c[6]) {
    float2* o = reinterpret_cast<float2*>(cov + row * 6);
    o[0] = make_float2(c[0], c[1]);
    o[1] = make_float2(c[2], c[3]);
    o[2] = make_float2(c[4], c[5]);
}

// ---------------------------------------------------------------------------
// Fast path (DESIGN.md §kNN fast path): ring 1 only, per-lane max-heap of K keys
// (d2 bits << 32 | sorted position) in shared memory (column per lane, so any
// slot index is bank-conflict free), sift-up while filling, replace-root +
// sift-down afterwards (O(log K) per accepted candidate instead of O(K) register
// shifts), one Batcher network sort at the end. Returns false -- the query is
// DEFERRED to the exact ring-expanding path -- when the stop rule needs ring 2,
// fewer than K candidates were found, or a d2 tie touches the result.
// ---------------------------------------------------------------------------
template <int KCAP>
__device__ __forceinline__ bool knn_fast(const float4* __restrict__ pts, const HashEntry* __restrict__ H,
                                         const Grid& g, const QGeom& G, int K, unsigned long long* __restrict__ Hl,
                                         unsigned long long (&L)[KCAP]) {
    int cnt = 0;
    unsigned long long top = 0ull;
    unsigned tie = 0xffffffffu;
    const float s = g.cell, slack = g.slack;
    const float lox = axis_gap(-1, G.fx, s, slack), hix = axis_gap(1, G.fx, s, slack);
    const float loy = axis_gap(-1, G.fy, s, slack), hiy = axis_gap(1, G.fy, s, slack);
    const float loz = axis_gap(-1, G.fz, s, slack), hiz = axis_gap(1, G.fz, s, slack);
#define HSLOT(i) Hl[(i) * kBlock]
    for (int c = 0; c < 27; ++c) {
        const int dx = c_off27[c][0], dy = c_off27[c][1], dz = c_off27[c][2];
        if (cnt == K) {
            const float gx = dx < 0 ? lox : (dx > 0 ? hix : 0.0f);
            const float gy = dy < 0 ? loy : (dy > 0 ? hiy : 0.0f);
            const float gz = dz < 0 ? loz : (dz > 0 ? hiz : 0.0f);
            const float lb2 = __fmaf_rn(gz, gz, __fmaf_rn(gy, gy, gx * gx));
            if (lb2 * kRel > __uint_as_float(hi32(top))) continue;
        }
        const int2 rng = cell_lookup(H, g, G.cx + dx, G.cy + dy, G.cz + dz);
        for (int j = rng.x; j < rng.y; ++j) {
            const float4 p = __ldg(pts + j);
            const unsigned hi = __float_as_uint(dist2(G.qx, G.qy, G.qz, p.x, p.y, p.z));
            const unsigned long long key = ((unsigned long long)hi << 32) | (unsigned)j;
            if (cnt < K) {  // fill: sift-up into the max-heap
                int i = cnt++;
                while (i > 0) {
                    const int par = (i - 1) >> 1;
                    const unsigned long long pv = HSLOT(par);
                    if (hi32(pv) >= hi) break;
                    HSLOT(i) = pv;
                    i = par;
                }
                HSLOT(i) = key;
                if (cnt == K) top = HSLOT(0);
            } else {
                const unsigned th = hi32(top);
                if (hi < th) {  // replace the root, sift down
                    int i = 0;
                    while (true) {
                        const int l = 2 * i + 1;
                        if (l >= K) break;
                        unsigned long long cv = HSLOT(l);
                        int ci = l;
                        if (l + 1 < K) {
                            const unsigned long long rv = HSLOT(l + 1);
                            if (hi32(rv) > hi32(cv)) {
                                cv = rv;
                                ci = l + 1;
                            }
                        }
                        if (hi32(cv) <= hi) break;
                        HSLOT(i) = cv;
                        i = ci;
                    }
                    HSLOT(i) = key;
                    top = HSLOT(0);
                    if (hi32(top) == th) tie = min(tie, th);  // evicted key tied with the new K-th
                } else if (hi == th) {
                    tie = min(tie, hi);  // rejected key tied with the K-th
                }
            }
        }
    }
    if (cnt < K) return false;
    // stop rule after the 27-voxel cube (R = 1)
    {
        const float mx = fminf(G.fx + s, 2.0f * s - G.fx);
        const float my = fminf(G.fy + s, 2.0f * s - G.fy);
        const float mz = fminf(G.fz + s, 2.0f * s - G.fz);
        const float m = fminf(mx, fminf(my, mz)) - slack;
        if (!(m > 0.0f && __uint_as_float(hi32(top)) < m * m * kRel)) return false;
    }
    if (tie == hi32(top)) return false;
#pragma unroll
    for (int r = 0; r < KCAP; ++r) L[r] = (r < K) ? HSLOT(r) : kEmptyKey;
#undef HSLOT
    sort_network<KCAP>(L);
    bool dup = false;
#pragma unroll
    for (int r = 0; r + 1 < KCAP; ++r)
        if (r + 1 < K) dup |= hi32(L[r]) == hi32(L[r + 1]);
    return !dup;
}

// rows from the fast path: slots 0..K-1 ascending, payload = sorted position
template <int KCAP>
__device__ __forceinline__ void emit_fast(const float4* __restrict__ pts, const unsigned long long (&L)[KCAP], int K,
                                          int64_t row, float eps, int32_t* __restrict__ nbr, float* __restrict__ d2,
                                          float* __restrict__ cov) {
    const float4 p0 = __ldg(pts + (unsigned)(L[0] & 0xffffffffu));
    float sx = 0.f, sy = 0.f, sz = 0.f;
#pragma unroll
    for (int r = 0; r < KCAP; ++r) {
        if (r >= K) continue;
        const float4 p = __ldg(pts + (unsigned)(L[r] & 0xffffffffu));
        if (nbr) nbr[row * K + r] = __float_as_int(p.w);
        if (d2) d2[row * K + r] = __uint_as_float(hi32(L[r]));
        sx += p.x - p0.x;
        sy += p.y - p0.y;
        sz += p.z - p0.z;
    }
    if (!cov) return;
    const float invk = 1.0f / (float)K;
    const float mx = sx * invk, my = sy * invk, mz = sz * invk;
    float c00 = 0.f, c01 = 0.f, c02 = 0.f, c11 = 0.f, c12 = 0.f, c22 = 0.f;
#pragma unroll
    for (int r = 0; r < KCAP; ++r) {
        if (r >= K) continue;
        const float4 p = __ldg(pts + (unsigned)(L[r] & 0xffffffffu));
        const float x = (p.x - p0.x) - mx, y = (p.y - p0.y) - my, z = (p.z - p0.z) - mz;
        c00 = fmaf(x, x, c00);
        c01 = fmaf(x, y, c01);
        c02 = fmaf(x, z, c02);
        c11 = fmaf(y, y, c11);
        c12 = fmaf(y, z, c12);
        c22 = fmaf(z, z, c22);
    }
    float c[6];
    plane_cov(c00 * invk, c01 * invk, c02 * invk, c11 * invk, c12 * invk, c22 * invk, eps, c);
    store_cov(cov, row, c);
}

__device__ __forceinline__ void push_warp(int* __restrict__ count, int* __restrict__ list, bool pred, int value) {
    const unsigned mask = __ballot_sync(0xffffffffu, pred);
    if (!pred) return;
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(mask) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(count, __popc(mask));
    base = __shfl_sync(mask, base, leader);
    list[base + __popc(mask & ((1u << lane) - 1))] = value;
}

// self queries: thread t handles sorted point t (fast path), deferring the rest
template <int KCAP>
__global__ void __launch_bounds__(kBlock) k_knn_self(const float4* __restrict__ pts, const HashEntry* __restrict__ H,
                                                     Grid g, int64_t n, int K, float eps, int32_t* __restrict__ nbr,
                                                     float* __restrict__ d2, float* __restrict__ cov,
                                                     int* __restrict__ def_count, int* __restrict__ def_list) {
    extern __shared__ unsigned long long heap[];
    const int64_t t = blockIdx.x * (int64_t)kBlock + threadIdx.x;
    bool defer = false;
    if (t < n) {
        const float4 q = __ldg(pts + t);
        const QGeom G = make_geom(g, q.x, q.y, q.z);
        unsigned long long L[KCAP];
        if (knn_fast<KCAP>(pts, H, g, G, K, heap + threadIdx.x, L))
            emit_fast<KCAP>(pts, L, K, __float_as_int(q.w), eps, nbr, d2, cov);
        else
            defer = true;
    }
    push_warp(def_count, def_list, defer, (int)t);
}

// external queries visited in voxel-sorted order (perm)
template <int KCAP>
__global__ void __launch_bounds__(kBlock) k_knn_ext(const float4* __restrict__ pts, const HashEntry* __restrict__ H,
                                                    Grid g, const float* __restrict__ q, const int* __restrict__ perm,
                                                    int64_t m, int K, int32_t* __restrict__ nbr,
                                                    float* __restrict__ d2, int* __restrict__ def_count,
                                                    int* __restrict__ def_list) {
    extern __shared__ unsigned long long heap[];
    const int64_t t = blockIdx.x * (int64_t)kBlock + threadIdx.x;
    bool defer = false;
    int row = 0;
    if (t < m) {
        row = perm[t];
        const float qx = q[3 * (int64_t)row], qy = q[3 * (int64_t)row + 1], qz = q[3 * (int64_t)row + 2];
        if (!(isfinite(qx) && isfinite(qy) && isfinite(qz))) {
            for (int r = 0; r < K; ++r) {
                nbr[(int64_t)row * K + r] = -1;
                d2[(int64_t)row * K + r] = __int_as_float(0x7f800000);
            }
        } else {
            const QGeom G = make_geom(g, qx, qy, qz);
            unsigned long long L[KCAP];
            if (knn_fast<KCAP>(pts, H, g, G, K, heap + threadIdx.x, L))
                emit_fast<KCAP>(pts, L, K, row, 0.f, nbr, d2, nullptr);
            else
                defer = true;
        }
    }
    push_warp(def_count, def_list, defer, row);
}

// Deferred queries (ring >= 2, too few candidates, or d2 ties): the exact
// ring-expanding search with (d2, original index) keys. self_mode: list holds
// sorted positions; else original query indices into qext.
template <int KCAP>
__global__ void __launch_bounds__(kBlock) k_knn_deferred(const float4* __restrict__ pts,
                                                         const float4* __restrict__ pts_orig,
                                                         const HashEntry* __restrict__ H, Grid g,
                                                         const float* __restrict__ qext, int self_mode,
                                                         const int* __restrict__ def_count,
                                                         const int* __restrict__ def_list, int K, float eps,
                                                         int32_t* __restrict__ nbr, float* __restrict__ d2,
                                                         float* __restrict__ cov, int* __restrict__ ovf_count,
                                                         int* __restrict__ ovf_list) {
    const int total = *def_count;
    for (int t = blockIdx.x * kBlock + threadIdx.x; t < total; t += gridDim.x * kBlock) {
        const int id = def_list[t];
        float qx, qy, qz;
        int64_t row;
        if (self_mode) {
            const float4 p = __ldg(pts + id);
            qx = p.x;
            qy = p.y;
            qz = p.z;
            row = __float_as_int(p.w);
        } else {
            qx = qext[3 * (int64_t)id];
            qy = qext[3 * (int64_t)id + 1];
            qz = qext[3 * (int64_t)id + 2];
            row = id;
        }
        const QGeom G = make_geom(g, qx, qy, qz);
        unsigned long long L[KCAP];
        unsigned tie_hi;
        int ovf;
        knn_search<KCAP, true>(pts, H, g, G, L, K, tie_hi, ovf);
        if (ovf) {
            ovf_list[atomicAdd(ovf_count, 1)] = id;
            continue;
        }
        write_row<KCAP, true>(pts, pts_orig, L, K, row, nbr, d2);
        if (cov) {
            float c[6];
            cov_row<KCAP, true>(pts, pts_orig, L, K, eps, c);
            store_cov(cov, row, c);
        }
    }
}

// Brute force for overflow queries: one block per query, exact (d2, orig) keys.
// Each thread keeps a sorted top-K of its strided share; the block then merges by
// K rounds of a min-reduction over the 256 list heads.
constexpr int kBFBlock = 256;
template <int KCAP>
__global__ void __launch_bounds__(kBFBlock) k_knn_bruteforce(const float4* __restrict__ pts,
                                                             const float4* __restrict__ pts_orig, int64_t n,
                                                             const float* __restrict__ qext, int self_mode,
                                                             const int* __restrict__ list,
                                                             const int* __restrict__ count, int K, float eps,
                                                             int32_t* __restrict__ nbr, float* __restrict__ d2,
                                                             float* __restrict__ cov) {
    if ((int)blockIdx.x >= *count) return;
    const int qi = list[blockIdx.x];
    float qx, qy, qz;
    int64_t row;
    if (self_mode) {
        const float4 p = pts[qi];
        qx = p.x;
        qy = p.y;
        qz = p.z;
        row = __float_as_int(p.w);
    } else {
        qx = qext[3 * (int64_t)qi];
        qy = qext[3 * (int64_t)qi + 1];
        qz = qext[3 * (int64_t)qi + 2];
        row = qi;
    }
    unsigned long long L[KCAP];
#pragma unroll
    for (int r = 0; r < KCAP; ++r) L[r] = (r < KCAP - K) ? 0ull : kEmptyKey;
    for (int64_t j = threadIdx.x; j < n; j += kBFBlock) {
        const float4 p = __ldg(pts + j);
        const float dd = dist2(qx, qy, qz, p.x, p.y, p.z);
        const unsigned long long key = ((unsigned long long)__float_as_uint(dd) << 32) | __float_as_uint(p.w);
        if (key < L[KCAP - 1]) topk_insert<KCAP>(L, key);
    }
    __shared__ unsigned long long heads[kBFBlock];
    __shared__ unsigned long long out[KCAP];
    int h = KCAP - K;  // next unconsumed slot of this thread's list
    for (int r = 0; r < K; ++r) {
        unsigned long long mine = kEmptyKey;
#pragma unroll
        for (int s = 0; s < KCAP; ++s)
            if (s == h) mine = L[s];
        heads[threadIdx.x] = mine;
        __syncthreads();
        for (int w = kBFBlock / 2; w > 0; w >>= 1) {
            if ((int)threadIdx.x < w) heads[threadIdx.x] = min(heads[threadIdx.x], heads[threadIdx.x + w]);
            __syncthreads();
        }
        const unsigned long long best = heads[0];
        if (mine == best && best != kEmptyKey) ++h;  // keys are unique (orig index)
        if (threadIdx.x == 0) out[r] = best;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        for (int r = 0; r < K; ++r) {
            if (nbr) nbr[row * K + r] = (int)(out[r] & 0xffffffffu);
            if (d2) d2[row * K + r] = __uint_as_float(hi32(out[r]));
        }
        if (cov) {
            // covariance through the original-order array (rare path)
            const float4 p0 = pts_orig[out[0] & 0xffffffffu];
            float sx = 0.f, sy = 0.f, sz = 0.f;
            for (int r = 0; r < K; ++r) {
                const float4 p = pts_orig[out[r] & 0xffffffffu];
                sx += p.x - p0.x;
                sy += p.y - p0.y;
                sz += p.z - p0.z;
            }
            const float invk = 1.0f / (float)K;
            const float mx = sx * invk, my = sy * invk, mz = sz * invk;
            float c00 = 0.f, c01 = 0.f, c02 = 0.f, c11 = 0.f, c12 = 0.f, c22 = 0.f;
            for (int r = 0; r < K; ++r) {
                const float4 p = pts_orig[out[r] & 0xffffffffu];
                const float x = (p.x - p0.x) - mx, y = (p.y - p0.y) - my, z = (p.z - p0.z) - mz;
                c00 = fmaf(x, x, c00);
                c01 = fmaf(x, y, c01);
                c02 = fmaf(x, z, c02);
                c11 = fmaf(y, y, c11);
                c12 = fmaf(y, z, c12);
                c22 = fmaf(z, z, c22);
            }
            float c[6];
            plane_cov(c00 * invk, c01 * invk, c02 * invk, c11 * invk, c12 * invk, c22 * invk, eps, c);
            store_cov(cov, row, c);
        }
    }
}

__global__ void k_query_keys(const float* __restrict__ q, int64_t m, Grid g, unsigned long long* __restrict__ keys,
                             int* __restrict__ vals) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= m) return;
    const float x = q[3 * i], y = q[3 * i + 1], z = q[3 * i + 2];
    unsigned long long key = kEmptyKey;
    if (isfinite(x) && isfinite(y) && isfinite(z)) {
        const int cx = min(max(cell_coord(x, g.ox, g.inv_cell), 0), g.nx - 1);
        const int cy = min(max(cell_coord(y, g.oy, g.inv_cell), 0), g.ny - 1);
        const int cz = min(max(cell_coord(z, g.oz, g.inv_cell), 0), g.nz - 1);
        key = cell_key(g, cx, cy, cz);
    }
    keys[i] = key;
    vals[i] = (int)i;
}

struct Scratch {
    void* p = nullptr;
    cudaStream_t s = nullptr;
    ~Scratch() {
        if (p) cudaFreeAsync(p, s);
    }
    int alloc(size_t bytes, cudaStream_t st) {
        s = st;
        if (cudaMallocAsync(&p, bytes ? bytes : 16, st) != cudaSuccess) {
            cudaGetLastError();
            return set_error(GICP_ENOMEM, "scratch allocation failed");
        }
        return GICP_OK;
    }
};

template <int KCAP>
int run_queries(const gicp_index_s* idx, const float* qext, const int* perm, int64_t m, int k, float eps,
                int32_t* nbr, float* d2, float* cov, cudaStream_t s) {
    Scratch lists;
    int rc;
    // [def_count, ovf_count, pad, pad] [def_list: m] [ovf_list: m]
    if ((rc = lists.alloc(sizeof(int) * (2 * m + 4), s))) return rc;
    int* def_count = (int*)lists.p;
    int* ovf_count = def_count + 1;
    int* def_list = def_count + 4;
    int* ovf_list = def_list + m;
    if ((rc = check_cuda(cudaMemsetAsync(def_count, 0, 4 * sizeof(int), s), "memset"))) return rc;
    const unsigned blocks = (unsigned)((m + kBlock - 1) / kBlock);
    const size_t shmem = (size_t)KCAP * kBlock * sizeof(unsigned long long);
    if (qext == nullptr) {
        k_knn_self<KCAP><<<blocks, kBlock, shmem, s>>>(idx->pts, idx->hash, idx->g, m, k, eps, nbr, d2, cov,
                                                        def_count, def_list);
    } else {
        k_knn_ext<KCAP><<<blocks, kBlock, shmem, s>>>(idx->pts, idx->hash, idx->g, qext, perm, m, k, nbr, d2,
                                                       def_count, def_list);
    }
    const unsigned dblocks = (unsigned)std::min<int64_t>(blocks, 148 * 16);
    k_knn_deferred<KCAP><<<dblocks, kBlock, 0, s>>>(idx->pts, idx->pts_orig, idx->hash, idx->g, qext,
                                                     qext == nullptr, def_count, def_list, k, eps, nbr, d2, cov,
                                                     ovf_count, ovf_list);
    const unsigned bf_blocks = (unsigned)std::min<int64_t>(m, 65535);
    k_knn_bruteforce<KCAP><<<bf_blocks, kBFBlock, 0, s>>>(idx->pts, idx->pts_orig, idx->n, qext, qext == nullptr,
                                                          ovf_list, ovf_count, k, eps, nbr, d2, cov);
    return check_cuda(cudaGetLastError(), "knn launch");
}

template <int KCAP>
int run_self(const gicp_index_s* idx, int k, float eps, int32_t* nbr, float* d2, float* cov, cudaStream_t s) {
    return run_queries<KCAP>(idx, nullptr, nullptr, idx->n, k, eps, nbr, d2, cov, s);
}

template <int KCAP>
int run_ext(const gicp_index_s* idx, const float* q, int64_t m, int k, int32_t* nbr, float* d2, cudaStream_t s) {
    Scratch keys_in, keys_out, vals_in, perm, temp;
    int rc;
    if ((rc = keys_in.alloc(m * 8, s)) || (rc = keys_out.alloc(m * 8, s)) || (rc = vals_in.alloc(m * 4, s)) ||
        (rc = perm.alloc(m * 4, s)))
        return rc;
    k_query_keys<<<(unsigned)((m + 255) / 256), 256, 0, s>>>(q, m, idx->g, (unsigned long long*)keys_in.p,
                                                              (int*)vals_in.p);
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, (unsigned long long*)keys_in.p, (unsigned long long*)keys_out.p,
                                    (int*)vals_in.p, (int*)perm.p, (int)m, 0, 64, s);
    if ((rc = temp.alloc(tb, s))) return rc;
    cub::DeviceRadixSort::SortPairs(temp.p, tb, (unsigned long long*)keys_in.p, (unsigned long long*)keys_out.p,
                                    (int*)vals_in.p, (int*)perm.p, (int)m, 0, 64, s);
    return run_queries<KCAP>(idx, q, (int*)perm.p, m, k, 0.f, nbr, d2, nullptr, s);
}

}  // namespace

#define GICP_KCAP_DISPATCH(K, CALL)       \
    switch ((K + 3) / 4) {                \
        case 1: { constexpr int KC = 4; return CALL; }  \
        case 2: { constexpr int KC = 8; return CALL; }  \
        case 3: { constexpr int KC = 12; return CALL; } \
        case 4: { constexpr int KC = 16; return CALL; } \
        case 5: { constexpr int KC = 20; return CALL; } \
        case 6: { constexpr int KC = 24; return CALL; } \
        case 7: { constexpr int KC = 28; return CALL; } \
        default: { constexpr int KC = 32; return CALL; } \
    }

int launch_knn_self(const gicp_index_s* idx, int k, float eps, int32_t* nbr, float* d2, float* cov, cudaStream_t s) {
    GICP_KCAP_DISPATCH(k, (run_self<KC>(idx, k, eps, nbr, d2, cov, s)));
}

int launch_knn(const gicp_index_s* idx, const float* q, int64_t m, int k, int32_t* nbr, float* d2, cudaStream_t s) {
    GICP_KCAP_DISPATCH(k, (run_ext<KC>(idx, q, m, k, nbr, d2, s)));
}

}  // namespace gicp
