// knn.cu -- exact kNN on the voxel pyramid, and the fused kNN + covariance kernel.
//
// Paper: "GPU-based nearest points search and covariance computation" (PAPER.md
// l.413, l.798); the CPU bottleneck it removes is "the corresponding points
// search" during covariance estimation (l.797, l.403-405).
//
// Definition (include/gicp.h, reading R9): for each query the k smallest
// keys (fp32 d2 in the fixed FMA order, ORIGINAL target index) over ALL targets.
//
// Design:
//  * fast path, one thread per query, queries in Morton order (a warp's 32 lanes
//    are a compact 3-D block): the 27 voxels of the query's level-l cube,
//    nearest-first, pruned by box distance; a per-lane max-heap of K keys
//    (bits(d2) << 32 | sorted position) in shared memory; heap updates are
//    PREDICATED and issued once per candidate step for the whole warp (no
//    per-lane divergent sift loops); a Batcher network sorts the K keys at the end.
//  * the stop rule (no unsearched point can beat the K-th key, conservative
//    slack) decides whether the 27-voxel cube sufficed; if not, the query moves to
//    the next pyramid level (cell x 2) -- sparse regions of a scan need few levels;
//  * queries whose result is touched by an exact d2 tie (where the definition
//    orders by ORIGINAL index, the fast path's payload is the sorted position), or
//    that exhaust the pyramid, go to the exact ring-expanding search with
//    (d2, original index) keys; pathological ones to a block brute force.
#include <cub/cub.cuh>

#include <cstdio>
#include <cstdlib>

#include "cov_device.cuh"
#include "gicp_internal.cuh"
#include "sortnet.cuh"

namespace gicp {
namespace {

constexpr int kBlock = 128;
#ifndef GICP_KNN_PROF
#define GICP_KNN_PROF 0  // diagnostics build: per-warp step/replacement counters
#endif
#if GICP_KNN_PROF
__device__ unsigned long long g_kprof[64];  // 16 counters per level 0, 1, 2, >= 3
#define KPROF(x) x
#else
#define KPROF(x)
#endif
#ifndef GICP_KNN_REGSORT
#define GICP_KNN_REGSORT 1  // sort the final K keys in registers
#endif
#ifndef GICP_KNN_MINB
#define GICP_KNN_MINB 6
#endif
constexpr int kMaxRing = 24;

__device__ __forceinline__ unsigned hi32(unsigned long long k) { return (unsigned)(k >> 32); }

// sorted register list insertion (exact path)
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

template <int N, bool FULL = false>
__device__ __forceinline__ void sort_network(unsigned long long (&v)[N]) {
    constexpr SortNet net = make_sortnet(N);
#pragma unroll
    for (int c = 0; c < net.n; ++c) {
        unsigned long long& a = v[net.a[c]];
        unsigned long long& b = v[net.b[c]];
        const bool sw = FULL ? b < a : hi32(b) < hi32(a);
        const unsigned long long t = a;
        a = sw ? b : a;
        b = sw ? t : b;
    }
}

// the same network on a shared-memory column (stride kBlock) -- keeps the K keys
// out of registers
template <int N, int STRIDE, bool FULL = false>
__device__ __forceinline__ void sort_network_smem(unsigned long long* __restrict__ H) {
    constexpr SortNet net = make_sortnet(N);
#pragma unroll
    for (int c = 0; c < net.n; ++c) {
        const unsigned long long a = H[net.a[c] * STRIDE], b = H[net.b[c] * STRIDE];
        if (FULL ? b < a : hi32(b) < hi32(a)) {
            H[net.a[c] * STRIDE] = b;
            H[net.b[c] * STRIDE] = a;
        }
    }
}

constexpr int floor_log2(int x) { return x <= 1 ? 0 : 1 + floor_log2(x / 2); }

// ---------------------------------------------------------------------------
// Exact path: ring-expanding search at one level with (d2, original index) keys,
// register-resident sorted list padded at the FRONT (K-th key = slot KCAP-1).
// ---------------------------------------------------------------------------
template <int KCAP>
__device__ __forceinline__ void knn_exact(const float4* __restrict__ pts, const Grid& g, const QGeom& G,
                                          unsigned long long (&L)[KCAP], int K, int& overflow) {
#pragma unroll
    for (int r = 0; r < KCAP; ++r) L[r] = (r < KCAP - K) ? 0ull : kEmptyKey;
    overflow = 0;
    const float s = g.cell, slack = g.slack;
    auto scan = [&](int2 rng) {
        for (int j = rng.x; j < rng.y; ++j) {
            const float4 p = __ldg(pts + j);
            const unsigned hi = __float_as_uint(dist2(G.qx, G.qy, G.qz, p.x, p.y, p.z));
            if (hi <= hi32(L[KCAP - 1])) {
                const unsigned long long key = ((unsigned long long)hi << 32) | __float_as_uint(p.w);
                if (key < L[KCAP - 1]) topk_insert<KCAP>(L, key);
            }
        }
    };
    const int R0 = max(max(max(-G.cx, G.cx - (g.nx - 1)), max(-G.cy, G.cy - (g.ny - 1))),
                       max(-G.cz, G.cz - (g.nz - 1)));  // rings below R0 lie outside the grid
    for (int R = 0;; ++R) {
        if (R > 1 && R < R0) R = R0;
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
                    if (lb2 * kRel > __uint_as_float(hi32(L[KCAP - 1]))) return;  // NaN (not full) -> false
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
        if (R == 0) continue;
        const float m = cube_margin(G, s, slack, R);
        if (m > 0.0f && __uint_as_float(hi32(L[KCAP - 1])) < m * m * kRel) break;
        const bool covers = G.cx - R <= 0 && G.cx + R >= g.nx - 1 && G.cy - R <= 0 && G.cy + R >= g.ny - 1 &&
                            G.cz - R <= 0 && G.cz + R >= g.nz - 1;
        if (covers) break;
    }
}

// ---------------------------------------------------------------------------
// Fast path at one level (warp-synchronous: every lane of the warp must call it;
// `active` = the lane has a query). Status: 0 done (L[0..K-1] ascending, payload =
// sorted position), 1 try the next level, 2 exact path (tie / too few points).
//
// Per lane: (A) the non-empty voxels of the 27-voxel cube, nearest-first, are
// gathered into a shared-memory range list (27 hash probes, fully unrolled so the
// probes overlap; neighbour Morton keys by dilated-integer arithmetic); (B) one
// flattened candidate stream over those ranges (the warp iterates max over lanes
// of the lane's candidate count, not the sum over voxels of per-voxel maxima);
// (C) a max-heap of K keys in shared memory, padded to a full binary tree of
// depth D with 0-keys so sift-down needs no bound checks; fill (sift-up) and
// replace-root (sift-down) are predicated and issued once per step for the warp.
// ---------------------------------------------------------------------------
constexpr unsigned long long kMortonX = 0x1249249249249249ull;  // dilated bits of x

__device__ __forceinline__ unsigned long long dil_inc(unsigned long long a, unsigned long long M) {
    return ((a | ~M) + 1ull) & M;
}
__device__ __forceinline__ unsigned long long dil_dec(unsigned long long a, unsigned long long M) {
    return (a - 1ull) & M;
}

template <int KCAP>
struct FastShape {
    static constexpr int D = floor_log2(KCAP);   // heap depth bound for K <= KCAP
    static constexpr int NH = (2 << D) - 1;      // full binary tree slots (>= KCAP)
};

// level-0 voxel adjacency lists of the index (index.cu)
struct AdjView {
    const int2* oc;
    const int2* rng;  // packed entries (adj_pack)
    const int2* oc1;  // level 1 (escalated queries)
    const int2* rng1;
};

template <int KCAP, bool EXACT = false>
__device__ __forceinline__ int knn_fast(const float4* __restrict__ pts, const Grid& g, const QGeom& G, int K,
                                        bool active, unsigned long long* __restrict__ Hl, AdjView adj) {
    constexpr int D = FastShape<KCAP>::D;
    const float s = g.cell, slack = g.slack;
#define HSLOT(i) Hl[(i) * kBlock]
    // (A) the voxel ranges: the index's adjacency list of the query's voxel when it
    // is occupied at level 0 (no probes, shared by the voxel's queries), else a
    // gather of the 27 probes into a thread-local list
    int2 rl[27];
    float lbl[27];
    int nr = 0;
    int a0 = 0, a1 = 0;
    bool use_adj = false;
    const int2* adj_oc = g.level == 0 ? adj.oc : (g.level == 1 ? adj.oc1 : nullptr);
    const int2* adj_rng = g.level == 0 ? adj.rng : adj.rng1;
    if (active && adj_oc != nullptr) {
        const int2 own = cell_lookup(g, G.cx, G.cy, G.cz);
        if (own.y > own.x) {
            use_adj = true;
            const int2 oc = __ldg(adj_oc + own.x);
            a0 = oc.x;
            a1 = oc.x + oc.y;
        }
    }
    if (active && !use_adj) {
        const float gxs[3] = {axis_gap(-1, G.fx, s, slack), 0.0f, axis_gap(1, G.fx, s, slack)};
        const float gys[3] = {axis_gap(-1, G.fy, s, slack), 0.0f, axis_gap(1, G.fy, s, slack)};
        const float gzs[3] = {axis_gap(-1, G.fz, s, slack), 0.0f, axis_gap(1, G.fz, s, slack)};
        const unsigned long long MX = kMortonX, MY = kMortonX << 1, MZ = kMortonX << 2;
        const unsigned long long kx = spread3((unsigned)G.cx), ky = spread3((unsigned)G.cy) << 1,
                                 kz = spread3((unsigned)G.cz) << 2;
        const unsigned long long kxs[3] = {dil_dec(kx, MX), kx, dil_inc(kx, MX)};
        const unsigned long long kys[3] = {dil_dec(ky, MY), ky, dil_inc(ky, MY)};
        const unsigned long long kzs[3] = {dil_dec(kz, MZ), kz, dil_inc(kz, MZ)};
        const bool okx[3] = {G.cx - 1 >= 0 && G.cx - 1 < g.nx, G.cx >= 0 && G.cx < g.nx, G.cx + 1 >= 0 && G.cx + 1 < g.nx};
        const bool oky[3] = {G.cy - 1 >= 0 && G.cy - 1 < g.ny, G.cy >= 0 && G.cy < g.ny, G.cy + 1 >= 0 && G.cy + 1 < g.ny};
        const bool okz[3] = {G.cz - 1 >= 0 && G.cz - 1 < g.nz, G.cz >= 0 && G.cz < g.nz, G.cz + 1 >= 0 && G.cz + 1 < g.nz};
#pragma unroll
        for (int c = 0; c < 27; ++c) {
            // nearest-first order: own, faces, edges, corners (same table as c_off27)
            constexpr signed char off[27][3] = {
                {0, 0, 0},   {-1, 0, 0},  {1, 0, 0},   {0, -1, 0},  {0, 1, 0},   {0, 0, -1},  {0, 0, 1},
                {-1, -1, 0}, {1, -1, 0},  {-1, 1, 0},  {1, 1, 0},   {-1, 0, -1}, {1, 0, -1},  {-1, 0, 1},
                {1, 0, 1},   {0, -1, -1}, {0, 1, -1},  {0, -1, 1},  {0, 1, 1},   {-1, -1, -1}, {1, -1, -1},
                {-1, 1, -1}, {1, 1, -1},  {-1, -1, 1}, {1, -1, 1},  {-1, 1, 1},  {1, 1, 1}};
            const int ix = off[c][0] + 1, iy = off[c][1] + 1, iz = off[c][2] + 1;
            if (!(okx[ix] && oky[iy] && okz[iz])) continue;
            const unsigned long long key = kxs[ix] | kys[iy] | kzs[iz];
            const int2 e = hash_find(g, key);
            if (e.y <= e.x) continue;  // voxel not occupied
            rl[nr] = e;
            lbl[nr] = __fmaf_rn(gzs[iz], gzs[iz], __fmaf_rn(gys[iy], gys[iy], gxs[ix] * gxs[ix]));
            ++nr;
        }
    }
    const float lox = axis_gap(-1, G.fx, s, slack), hix = axis_gap(1, G.fx, s, slack);
    const float loy = axis_gap(-1, G.fy, s, slack), hiy = axis_gap(1, G.fy, s, slack);
    const float loz = axis_gap(-1, G.fz, s, slack), hiz = axis_gap(1, G.fz, s, slack);
    // (B)+(C) flattened stream into the heap
    int cnt = 0;
    unsigned long long top = 0ull;  // root (max) once cnt == K
    unsigned tie = 0xffffffffu;
    // predicated replace-root + sift-down (padding slots hold 0-keys), issued once for the warp
    auto sift = [&](const bool repl, const unsigned long long key, const unsigned th) {
        const unsigned hi = hi32(key);
        int i = 0;
        bool moving = repl;
#pragma unroll
        for (int lev = 0; lev < D; ++lev) {
            const int l = 2 * i + 1;
            unsigned long long cv, rv;
            if (moving) {
                cv = HSLOT(l);
                rv = HSLOT(l + 1);
            }
            const bool pr = EXACT ? rv > cv : hi32(rv) > hi32(cv);
            const unsigned long long ch = pr ? rv : cv;
            const bool mv = moving && (EXACT ? ch > key : hi32(ch) > hi);
            if (mv) HSLOT(i) = ch;
            i = mv ? l + (int)pr : i;
            moving = mv;
        }
        if (repl) {
            HSLOT(i) = key;
            top = HSLOT(0);
            if (!EXACT && hi32(top) == th) tie = th;  // evicted key tied with the new K-th
        }
    };
    // one candidate step for the whole warp (lanes without a candidate idle)
    KPROF(unsigned p_steps = 0; unsigned p_fill = 0; unsigned p_repl = 0; unsigned p_lrepl = 0; unsigned p_cand = 0;
          unsigned p_ent = 0; unsigned p_adv = 0;)
    auto step = [&](const bool has, const int j, const float4 p) {
        unsigned hi = 0xffffffffu, pay = 0u;
        if (has) {
            hi = __float_as_uint(dist2(G.qx, G.qy, G.qz, p.x, p.y, p.z));
            pay = EXACT ? __float_as_uint(p.w) : (unsigned)j;
        }
        const unsigned long long key = ((unsigned long long)hi << 32) | pay;
        const bool fill = has && cnt < K;
        const unsigned th = hi32(top);
        // top == 0 until the heap is full and an idle lane has hi = ~0, so neither
        // needs its own test. A recorded tie value is the K-th at that time, which
        // never increases: the last one recorded is the smallest.
        const bool repl = EXACT ? (has && cnt == K && key < top) : hi < th;
        if (!EXACT && hi == th) tie = hi;  // rejected key tied with the K-th
        KPROF(p_steps++; p_fill += __any_sync(0xffffffffu, fill); p_repl += __any_sync(0xffffffffu, repl);
              p_lrepl += repl; p_cand += has;)
        if (__any_sync(0xffffffffu, fill)) {
            // predicated sift-up from slot cnt
            int i = cnt;
            bool moving = fill;
#pragma unroll
            for (int lev = 0; lev < D; ++lev) {
                const int par = (i - 1) >> 1;
                const bool can = moving && i > 0;
                unsigned long long pv = 0ull;
                if (can) pv = HSLOT(par);
                const bool mv = can && (EXACT ? pv < key : hi32(pv) < hi);
                if (mv) HSLOT(i) = pv;
                i = mv ? par : i;
                moving = mv;
            }
            if (fill) {
                HSLOT(i) = key;
                ++cnt;
                if (cnt == K) top = HSLOT(0);
            }
        }
        if (__any_sync(0xffffffffu, repl)) sift(repl, key, th);
        };
    int ri = use_adj ? a0 : 0;
    const int rend = use_adj ? a1 : nr;
    int pos = 0, end = 0;
    // software pipeline: the next adjacency entry and the next candidate point are
    // loaded one advance / one step ahead, so their latency overlaps the heap work
    int2 ne = make_int2(0, 0);
    if (use_adj && ri < rend) ne = __ldg(adj_rng + ri);
    float4 pn = make_float4(0.f, 0.f, 0.f, 0.f);
    while (true) {
        // advance exhausted lanes to their next non-pruned range
        KPROF(const unsigned e0 = p_ent;)
        while (pos == end && ri < rend) {
            KPROF(p_ent++;)
            int2 r;
            float lb2;
            if (use_adj) {
                const int2 e = ne;
                if (ri + 1 < rend) ne = __ldg(adj_rng + ri + 1);
                r = adj_range(e);
                lb2 = adj_lb2((unsigned)e.y, lox, hix, loy, hiy, loz, hiz);
            } else {
                r = rl[ri];
                lb2 = lbl[ri];
            }
            ++ri;
            if (cnt == K && lb2 * kRel > __uint_as_float(hi32(top))) continue;
            pos = r.x;
            end = r.y;
            pn = __ldg(pts + pos);
        }
        KPROF(p_adv += __reduce_max_sync(0xffffffffu, p_ent - e0);)
        const bool has = pos < end;
        if (!__any_sync(0xffffffffu, has)) break;
        const float4 p = pn;
        if (pos + 1 < end) pn = __ldg(pts + pos + 1);
        step(has, pos, p);
        if (has) ++pos;
    }
#if GICP_KNN_PROF
    if (!EXACT) {
        const unsigned full = 0xffffffffu;
        const unsigned v[9] = {p_steps, p_fill, p_repl, __reduce_add_sync(full, p_lrepl), __reduce_max_sync(full, p_lrepl),
                               __reduce_add_sync(full, p_cand), __reduce_add_sync(full, p_ent), p_adv,
                               (unsigned)__popc(__ballot_sync(full, active))};
        if ((threadIdx.x & 31) == 0) {
            const int b = 16 * min(g.level, 3);
            for (int i = 0; i < 8; ++i) atomicAdd(&g_kprof[b + i], (unsigned long long)v[i]);
            atomicAdd(&g_kprof[b + 8], 1ull);
            atomicAdd(&g_kprof[b + 9], (unsigned long long)v[8]);
        }
    }
#endif
    if (!active) return 0;
    if (cnt < K) return 1;
    const float m = cube_margin(G, s, slack, 1);
    if (!(m > 0.0f && __uint_as_float(hi32(top)) < m * m * kRel)) return 1;
    if (!EXACT && tie == hi32(top)) return 2;
    // sort the K keys in place (slots K..KCAP-1 temporarily +inf; the caller
    // restores the 0-key padding after emitting the row)
#if GICP_KNN_REGSORT
    {
        // the K keys through registers: the network's compare-exchanges are ALU
        // selects instead of dependent shared-memory round trips
        unsigned long long kk[KCAP];
#pragma unroll
        for (int r = 0; r < KCAP; ++r) kk[r] = r < K ? HSLOT(r) : kEmptyKey;
        sort_network<KCAP, EXACT>(kk);
#pragma unroll
        for (int r = 0; r < KCAP; ++r) HSLOT(r) = kk[r];
    }
#else
    for (int r = K; r < KCAP; ++r) HSLOT(r) = kEmptyKey;
    sort_network_smem<KCAP, kBlock, EXACT>(Hl);
#endif
    if (EXACT) return 0;
    bool dup = false;
    unsigned prev = hi32(HSLOT(0));
    for (int r = 1; r < K; ++r) {
        const unsigned h = hi32(HSLOT(r));
        dup |= h == prev;
        prev = h;
    }
#undef HSLOT
    return dup ? 2 : 0;
}

__device__ __forceinline__ void store_cov(float* cov, int64_t row, const float c[6]) {
    float2* o = reinterpret_cast<float2*>(cov + row * 6);
    o[0] = make_float2(c[0], c[1]);
    o[1] = make_float2(c[2], c[3]);
    o[2] = make_float2(c[4], c[5]);
}

// Emit one row from a list of K sorted positions (slots base..base+K-1 of L):
// nbr = original indices, d2, and the covariance of the K neighbours (two passes,
// fp32, relative to the first neighbour; eigen problem in fp64, cov_device.cuh).
template <int KCAP>
__device__ __forceinline__ void emit_row(const float4* __restrict__ pts, const unsigned long long (&L)[KCAP], int K,
                                         int base, bool spos_payload, const float4* __restrict__ pts_orig,
                                         int64_t row, float eps, int32_t* __restrict__ nbr, float* __restrict__ d2,
                                         float* __restrict__ cov) {
    auto pos = [&](unsigned long long key) -> int {
        const unsigned pay = (unsigned)(key & 0xffffffffu);
        return spos_payload ? (int)pay : __float_as_int(__ldg(pts_orig + pay).w);
    };
    unsigned long long first = 0ull;
#pragma unroll
    for (int r = 0; r < KCAP; ++r)
        if (r == base) first = L[r];
    const float4 p0 = __ldg(pts + pos(first));
    float sx = 0.f, sy = 0.f, sz = 0.f;
#pragma unroll
    for (int r = 0; r < KCAP; ++r) {
        if (r < base || r >= base + K) continue;
        const float4 p = __ldg(pts + pos(L[r]));
        if (nbr) nbr[row * K + (r - base)] = __float_as_int(p.w);
        if (d2) d2[row * K + (r - base)] = __uint_as_float(hi32(L[r]));
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
        if (r < base || r >= base + K) continue;
        const float4 p = __ldg(pts + pos(L[r]));
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

// emit a fast-path row: keys sorted ascending in the smem column Hl[0..K-1]
template <bool EXACT = false>
__device__ __forceinline__ void emit_row_smem(const float4* __restrict__ pts, const unsigned long long* __restrict__ Hl,
                                              int K, int64_t row, float eps, int32_t* __restrict__ nbr,
                                              float* __restrict__ d2, float* __restrict__ cov,
                                              const float4* __restrict__ pts_orig = nullptr) {
    // payload: sorted position (fast path) or original index (EXACT: map back)
    auto sp = [&](unsigned long long key) -> unsigned {
        const unsigned pay = (unsigned)(key & 0xffffffffu);
        return EXACT ? (unsigned)__float_as_int(__ldg(pts_orig + pay).w) : pay;
    };
    const float4 p0 = __ldg(pts + sp(Hl[0]));
    float sx = 0.f, sy = 0.f, sz = 0.f;
    for (int r = 0; r < K; ++r) {
        const unsigned long long key = Hl[r * kBlock];
        const float4 p = __ldg(pts + sp(key));
        if (nbr) nbr[row * K + r] = __float_as_int(p.w);
        if (d2) d2[row * K + r] = __uint_as_float(hi32(key));
        sx += p.x - p0.x;
        sy += p.y - p0.y;
        sz += p.z - p0.z;
    }
    if (!cov) return;
    const float invk = 1.0f / (float)K;
    const float mx = sx * invk, my = sy * invk, mz = sz * invk;
    float c00 = 0.f, c01 = 0.f, c02 = 0.f, c11 = 0.f, c12 = 0.f, c22 = 0.f;
    for (int r = 0; r < K; ++r) {
        const float4 p = __ldg(pts + sp(Hl[r * kBlock]));
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

// warp-aggregated append of `value` to list (lanes with pred)
__device__ __forceinline__ void push_warp(int* __restrict__ count, int* __restrict__ list, bool pred, int value) {
    const unsigned mask = __ballot_sync(0xffffffffu, pred);
    if (!mask) return;
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(mask) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(count, __popc(mask));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (pred) list[base + __popc(mask & ((1u << lane) - 1))] = value;
}

__device__ __forceinline__ void push_warp2(int* __restrict__ count, int2* __restrict__ list, bool pred, int2 value) {
    const unsigned mask = __ballot_sync(0xffffffffu, pred);
    if (!mask) return;
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(mask) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(count, __popc(mask));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (pred) list[base + __popc(mask & ((1u << lane) - 1))] = value;
}

struct Levels {
    Grid lv[kMaxLevels];
};

#include "knn_tile.cuh"

// the tiled level-0 stage for self queries (knn_tile.cuh): K = 10 and 20 (the
// configs' k); returns false when it does not apply (then the per-query kernel runs)
bool launch_tile(const gicp_index_s* idx, int k, float eps, int32_t* nbr, float* d2, float* cov, int* counts,
                 int* listA, int* listB, int2* exact, cudaStream_t s, const float* qext = nullptr,
                 const int* perm = nullptr, int64_t m = 0) {
    static const bool off = getenv("GICP_KNN_TILE") && atoi(getenv("GICP_KNN_TILE")) == 0;
    if (off || idx->tiles1 == nullptr || idx->tile_of == nullptr || idx->n == 0) return false;
    // the staged boxes pay off on dense, even clouds (the C3 map: ~35 points per
    // level-1 voxel); sparse, uneven ones (a scan's 1/r^2 falloff) run per query
    if (idx->n < 24 * idx->n_tiles1) return false;
    if (qext) {  // external queries in their cell-sorted order (perm)
        if (!perm || m <= 0 || (k != 10 && k != 20 && k != 32)) return false;
        const unsigned grid = (unsigned)((m + kTB - 1) / kTB);
#define GICP_TILE_EXT(KK)                                                                                         \
    k_knn_tile<KK, false, true><<<grid, kTB, 0, s>>>(idx->pts, idx->lv[0], idx->tiles1, idx->tile_of, m, eps, nbr, \
                                                     d2, nullptr, counts + 2, listA, counts + 0, exact, counts + 3,  \
                                                     listB, qext, perm)
        if (k == 32) GICP_TILE_EXT(32);
        else if (k == 20) GICP_TILE_EXT(20);
        else GICP_TILE_EXT(10);
#undef GICP_TILE_EXT
        return true;
    }
    if (perm || (k != 10 && k != 20)) return false;
    const unsigned grid = (unsigned)((idx->n + kTB - 1) / kTB);
    static const bool rows = getenv("GICP_KNN_ROWS") && atoi(getenv("GICP_KNN_ROWS")) == 1;
#define GICP_TILE_LAUNCH(KK, RR)                                                                                  \
    k_knn_tile<KK, RR><<<grid, kTB, 0, s>>>(idx->pts, idx->lv[0], idx->tiles1, idx->tile_of, idx->n, eps, nbr, d2, \
                                            cov, counts + 2, listA, counts + 0, exact, counts + 3, listB)
    if (k == 20) {
        if (rows) GICP_TILE_LAUNCH(20, true); else GICP_TILE_LAUNCH(20, false);
    } else {
        if (rows) GICP_TILE_LAUNCH(10, true); else GICP_TILE_LAUNCH(10, false);
    }
#undef GICP_TILE_LAUNCH
    return true;
}

// Query sources: self mode -> id = sorted position (xyz from pts, row = orig);
// external -> id = original query index into q.
struct QuerySrc {
    const float4* pts;
    const float* q;  // nullptr in self mode
    __device__ __forceinline__ void get(int id, float& x, float& y, float& z, int64_t& row) const {
        if (q == nullptr) {
            const float4 p = __ldg(pts + id);
            x = p.x;
            y = p.y;
            z = p.z;
            row = __float_as_int(p.w);
        } else {
            x = q[3 * (int64_t)id];
            y = q[3 * (int64_t)id + 1];
            z = q[3 * (int64_t)id + 2];
            row = id;
        }
    }
};

// One pyramid level of the fast path. Queries: ids = in_list[0 .. *in_count) or,
// when in_list == nullptr, the identity / perm over [0, m). Warp-uniform
// grid-stride loop (all 32 lanes stay together for the warp votes).
template <int KCAP>
__global__ void __launch_bounds__(kBlock, GICP_KNN_MINB) k_knn_level(QuerySrc src, AdjView adj, Grid g, const int* __restrict__ perm, int64_t m,
                                                      const int* __restrict__ in_list, const int* __restrict__ in_count,
                                                      int K, float eps, int32_t* __restrict__ nbr,
                                                      float* __restrict__ d2, float* __restrict__ cov,
                                                      int* __restrict__ next_count, int* __restrict__ next_list,
                                                      int* __restrict__ exact_count, int2* __restrict__ exact_list,
                                                      int last_level) {
    extern __shared__ unsigned long long smem[];
    constexpr int NH = FastShape<KCAP>::NH;
    unsigned long long* heap = smem;                                   // [NH][kBlock]
    for (int i = K; i < NH; ++i) heap[i * kBlock + threadIdx.x] = 0ull;  // 0-key padding of the full tree
    const int64_t total = in_list ? (int64_t)*in_count : m;
    const int lane = threadIdx.x & 31;
    const int64_t warp0 = ((int64_t)blockIdx.x * kBlock + (threadIdx.x & ~31));
    const int64_t stride = (int64_t)gridDim.x * kBlock;
    for (int64_t base = warp0; base < total; base += stride) {
        const int64_t t = base + lane;
        const bool active = t < total;
        int id = 0;
        float qx = 0.f, qy = 0.f, qz = 0.f;
        int64_t row = 0;
        bool finite = true;
        if (active) {
            id = in_list ? in_list[t] : (perm ? perm[t] : (int)t);
            src.get(id, qx, qy, qz, row);
            finite = isfinite(qx) && isfinite(qy) && isfinite(qz);
        }
        if (active && !finite) {  // external queries only (the index is finite)
            for (int r = 0; r < K; ++r) {
                nbr[row * K + r] = -1;
                d2[row * K + r] = __int_as_float(0x7f800000);
            }
        }
        const bool run = active && finite;
        const QGeom G = make_geom(g, qx, qy, qz);
        const int st = knn_fast<KCAP>(src.pts, g, G, K, run, heap + threadIdx.x, adj);
        if (run && st == 0) emit_row_smem(src.pts, heap + threadIdx.x, K, row, eps, nbr, d2, cov);
        for (int r = K; r < NH; ++r) heap[r * kBlock + threadIdx.x] = 0ull;  // restore the 0-key padding
        const bool to_next = run && st == 1 && !last_level;
        const bool to_exact = run && (st == 2 || (st == 1 && last_level));
        push_warp(next_count, next_list, to_next, id);
        push_warp2(exact_count, exact_list, to_exact, make_int2(id, g.level));
    }
}

// Queries level 0 could not settle climb the pyramid in ONE launch: each warp
// takes 32 of them through levels 1..L-1 (warp-synchronous fast path at every
// level, lanes that finish idle); still-unsettled queries and ties go to the
// exact path with the level they stopped at.
template <int KCAP>
__global__ void __launch_bounds__(kBlock, GICP_KNN_MINB) k_knn_escalate(QuerySrc src, AdjView adj, Levels lvs, int n_levels,
                                                                      const int* __restrict__ in_list,
                                                                      const int* __restrict__ in_count, int K,
                                                                      float eps, int32_t* __restrict__ nbr,
                                                                      float* __restrict__ d2, float* __restrict__ cov,
                                                                      int* __restrict__ exact_count,
                                                                      int2* __restrict__ exact_list) {
    extern __shared__ unsigned long long smem[];
    constexpr int NH = FastShape<KCAP>::NH;
    unsigned long long* heap = smem;
    for (int i = K; i < NH; ++i) heap[i * kBlock + threadIdx.x] = 0ull;
    const int64_t total = *in_count;
    const int lane = threadIdx.x & 31;
    const int64_t warp0 = ((int64_t)blockIdx.x * kBlock + (threadIdx.x & ~31));
    const int64_t stride = (int64_t)gridDim.x * kBlock;
    for (int64_t base = warp0; base < total; base += stride) {
        const int64_t t = base + lane;
        const bool active = t < total;
        int id = 0;
        float qx = 0.f, qy = 0.f, qz = 0.f;
        int64_t row = 0;
        if (active) {
            id = in_list[t];
            src.get(id, qx, qy, qz, row);
        }
        bool pending = active;
        int stop_level = n_levels - 1;
        bool to_exact = false;
        for (int l = 1; l < n_levels; ++l) {
            if (!__any_sync(0xffffffffu, pending)) break;
            const Grid g = lvs.lv[l];
            const QGeom G = make_geom(g, qx, qy, qz);
            const int st = knn_fast<KCAP>(src.pts, g, G, K, pending, heap + threadIdx.x, adj);
            if (pending && st == 0) emit_row_smem(src.pts, heap + threadIdx.x, K, row, eps, nbr, d2, cov);
            for (int r = K; r < NH; ++r) heap[r * kBlock + threadIdx.x] = 0ull;
            if (pending && st == 2) {
                to_exact = true;
                stop_level = l;
            }
            if (pending && st != 1) pending = false;
        }
        if (pending) to_exact = true;  // exhausted the pyramid: ring expansion at the last level
        push_warp2(exact_count, exact_list, to_exact, make_int2(id, stop_level));
    }
}

// Exact path for the rare queries the fast path could not settle (a d2 tie
// touching the result, or the pyramid exhausted): the same warp-synchronous heap
// search with (d2, ORIGINAL index) keys -- the definition's key, so ties need no
// special care -- from the level the query stopped at, climbing the pyramid; a
// query that exhausts it gets the ring-expanding search (register list).
template <int KCAP>
__global__ void __launch_bounds__(kBlock, GICP_KNN_MINB) k_knn_exact(QuerySrc src, AdjView adj, const float4* __restrict__ pts_orig,
                                                                   Levels lvs, int n_levels,
                                                                   const int2* __restrict__ list,
                                                                   const int* __restrict__ count, int K, float eps,
                                                                   int32_t* __restrict__ nbr, float* __restrict__ d2,
                                                                   float* __restrict__ cov, int* __restrict__ ovf_count,
                                                                   int* __restrict__ ovf_list) {
    extern __shared__ unsigned long long smem[];
    constexpr int NH = FastShape<KCAP>::NH;
    unsigned long long* heap = smem;
    for (int i = K; i < NH; ++i) heap[i * kBlock + threadIdx.x] = 0ull;
    const int64_t total = *count;
    const int lane = threadIdx.x & 31;
    // few entries (the usual case): one query per warp (lane 0) so they run in
    // parallel rather than as one warp's 32 lanes back to back
    const int64_t nwarps = (int64_t)gridDim.x * (kBlock / 32);
    const bool sparse = total <= nwarps;
    const int64_t wid = (int64_t)blockIdx.x * (kBlock / 32) + (threadIdx.x >> 5);
    const int64_t warp0 = sparse ? wid : ((int64_t)blockIdx.x * kBlock + (threadIdx.x & ~31));
    const int64_t stride = sparse ? nwarps : (int64_t)gridDim.x * kBlock;
    for (int64_t base = warp0; base < total; base += stride) {
        const int64_t t = sparse ? base : base + lane;
        const bool active = sparse ? (lane == 0) : (t < total);
        int2 e = make_int2(0, 0);
        float qx = 0.f, qy = 0.f, qz = 0.f;
        int64_t row = 0;
        if (active) {
            e = list[t];
            src.get(e.x, qx, qy, qz, row);
        }
        bool pending = active;
        for (int l = 0; l < n_levels; ++l) {
            const bool part = pending && l >= e.y;
            if (!__any_sync(0xffffffffu, part)) continue;
            const Grid g = lvs.lv[l];
            const QGeom G = make_geom(g, qx, qy, qz);
            const int st = knn_fast<KCAP, true>(src.pts, g, G, K, part, heap + threadIdx.x, adj);
            if (part && st == 0) {
                emit_row_smem<true>(src.pts, heap + threadIdx.x, K, row, eps, nbr, d2, cov, pts_orig);
                pending = false;
            }
            for (int r = K; r < NH; ++r) heap[r * kBlock + threadIdx.x] = 0ull;
        }
        if (pending) {  // pyramid exhausted: ring expansion at the last level (per lane)
            const Grid& g = lvs.lv[n_levels - 1];
            const QGeom G = make_geom(g, qx, qy, qz);
            unsigned long long L[KCAP];
            int ovf;
            knn_exact<KCAP>(src.pts, g, G, L, K, ovf);
            if (ovf)
                ovf_list[atomicAdd(ovf_count, 1)] = e.x;
            else
                emit_row<KCAP>(src.pts, L, K, KCAP - K, false, pts_orig, row, eps, nbr, d2, cov);
        }
    }
}

// Brute force for overflow queries: one block per query, exact (d2, orig) keys.
// Each thread keeps a sorted top-K of its strided share; the block then merges by
// K rounds of a min-reduction over the 256 list heads.
constexpr int kBFBlock = 256;
template <int KCAP>
__global__ void __launch_bounds__(kBFBlock) k_knn_bruteforce(QuerySrc src, const float4* __restrict__ pts_orig,
                                                             int64_t n, const int* __restrict__ list,
                                                             const int* __restrict__ count, int K, float eps,
                                                             int32_t* __restrict__ nbr, float* __restrict__ d2,
                                                             float* __restrict__ cov) {
    __shared__ unsigned long long heads[kBFBlock];
    __shared__ unsigned long long outk[KCAP];
    const int total = *count;
    for (int b = blockIdx.x; b < total; b += gridDim.x) {
        const int id = list[b];
        float qx, qy, qz;
        int64_t row;
        src.get(id, qx, qy, qz, row);
        unsigned long long L[KCAP];
#pragma unroll
        for (int r = 0; r < KCAP; ++r) L[r] = (r < KCAP - K) ? 0ull : kEmptyKey;
        for (int64_t j = threadIdx.x; j < n; j += kBFBlock) {
            const float4 p = __ldg(src.pts + j);
            const float dd = dist2(qx, qy, qz, p.x, p.y, p.z);
            const unsigned long long key = ((unsigned long long)__float_as_uint(dd) << 32) | __float_as_uint(p.w);
            if (key < L[KCAP - 1]) topk_insert<KCAP>(L, key);
        }
        int h = KCAP - K;  // next unconsumed slot of this thread's list
        for (int r = 0; r < K; ++r) {
            unsigned long long mine = kEmptyKey;
#pragma unroll
            for (int s2 = 0; s2 < KCAP; ++s2)
                if (s2 == h) mine = L[s2];
            heads[threadIdx.x] = mine;
            __syncthreads();
            for (int w = kBFBlock / 2; w > 0; w >>= 1) {
                if ((int)threadIdx.x < w) heads[threadIdx.x] = min(heads[threadIdx.x], heads[threadIdx.x + w]);
                __syncthreads();
            }
            const unsigned long long best = heads[0];
            if (mine == best && best != kEmptyKey) ++h;  // keys are unique (orig index)
            if (threadIdx.x == 0) outk[r] = best;
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            unsigned long long Lo[KCAP];
#pragma unroll
            for (int r = 0; r < KCAP; ++r) Lo[r] = outk[r < K ? r : K - 1];
            emit_row<KCAP>(src.pts, Lo, K, 0, false, pts_orig, row, eps, nbr, d2, cov);
        }
        __syncthreads();
    }
}

__global__ void k_query_keys(const float* __restrict__ q, int64_t m, Grid g, unsigned long long empty,
                             unsigned long long* __restrict__ keys, int* __restrict__ vals) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= m) return;
    const float x = q[3 * i], y = q[3 * i + 1], z = q[3 * i + 2];
    unsigned long long key = empty;  // non-finite queries last
    if (isfinite(x) && isfinite(y) && isfinite(z)) {
        const int cx = min(max(cell_coord(x, g.ox, g.inv_cell), 0), g.nx - 1);
        const int cy = min(max(cell_coord(y, g.oy, g.inv_cell), 0), g.ny - 1);
        const int cz = min(max(cell_coord(z, g.oz, g.inv_cell), 0), g.nz - 1);
        key = cell_key(cx, cy, cz);
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
            p = nullptr;
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
    // counts[16] | listA[m] | listB[m] | ovf[m] | exact[m] (int2)
    if ((rc = lists.alloc(sizeof(int) * (5 * m + 18), s))) return rc;
    int* counts = (int*)lists.p;
    int* listA = counts + 16;
    int* listB = listA + m;
    int* ovf = listB + m;
    int2* exact = reinterpret_cast<int2*>(ovf + m + (m & 1));
    if ((rc = check_cuda(cudaMemsetAsync(counts, 0, 16 * sizeof(int), s), "memset"))) return rc;
    const QuerySrc src{idx->pts, qext};
    const size_t shmem = (size_t)FastShape<KCAP>::NH * kBlock * sizeof(unsigned long long);
    cudaFuncSetAttribute(k_knn_level<KCAP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shmem);
    cudaFuncSetAttribute(k_knn_escalate<KCAP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shmem);
    cudaFuncSetAttribute(k_knn_exact<KCAP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shmem);
    const int L = idx->n_levels;
    const unsigned full_blocks = (unsigned)((m + kBlock - 1) / kBlock);
    const unsigned some_blocks = (unsigned)std::min<int64_t>(full_blocks, 148 * 8);
    Levels lvs;
    for (int l = 0; l < kMaxLevels; ++l) lvs.lv[l] = idx->lv[l < L ? l : L - 1];
    // level 0 over every query, then one launch that climbs the pyramid for the rest
    const AdjView adj{idx->adj_oc, idx->adj_rng, idx->adj_oc1, idx->adj_rng1};
    if (L > 1 && launch_tile(idx, k, eps, nbr, d2, cov, counts, listA, listB, exact, s, qext, perm, m)) {
        // tiles too dense to stage: the per-query level-0 kernel over their points
        k_knn_level<KCAP><<<some_blocks, kBlock, shmem, s>>>(src, adj, idx->lv[0], nullptr, m, listB, counts + 3, k, eps,
                                                             nbr, d2, cov, counts + 2, listA, counts + 0, exact, 0);
    } else {
        k_knn_level<KCAP><<<full_blocks, kBlock, shmem, s>>>(src, adj, idx->lv[0], perm, m, nullptr, nullptr, k, eps, nbr,
                                                             d2, cov, counts + 2, listA, counts + 0, exact, L == 1);
    }
    if (L > 1)
        k_knn_escalate<KCAP><<<some_blocks, kBlock, shmem, s>>>(src, adj, lvs, L, listA, counts + 2, k, eps, nbr, d2, cov,
                                                                counts + 0, exact);
    k_knn_exact<KCAP><<<some_blocks, kBlock, shmem, s>>>(src, adj, idx->pts_orig, lvs, L, exact, counts + 0, k, eps, nbr,
                                                          d2, cov, counts + 1, ovf);
    k_knn_bruteforce<KCAP><<<(unsigned)std::min<int64_t>(m, 1024), kBFBlock, 0, s>>>(
        src, idx->pts_orig, idx->n, ovf, counts + 1, k, eps, nbr, d2, cov);
    if (getenv("GICP_DEBUG_STATS")) {  // diagnostics only: path counts of this call
        int h[4] = {0, 0, 0, 0};
        cudaMemcpyAsync(h, counts, sizeof(h), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
#if GICP_KNN_PROF
        unsigned long long pv[64];
        cudaMemcpyFromSymbol(pv, g_kprof, sizeof(pv));
        for (int lv = 0; lv < 4; ++lv) {
            const unsigned long long* q = pv + 16 * lv;
            const double w = q[8] ? (double)q[8] : 1.0;
            if (!q[8]) continue;
            fprintf(stderr, "[gicp knn prof] level %d%s warp calls=%.0f active lanes/call %.1f | per call: steps %.1f "
                    "fill-steps %.1f repl-steps %.1f lane-repl %.1f max-lane-repl %.1f lane-cand %.1f lane-entries %.1f "
                    "adv-iters %.1f\n", lv, lv == 3 ? "+" : "", w, q[9] / w, q[0] / w, q[1] / w, q[2] / w, q[3] / w,
                    q[4] / w, q[5] / w, q[6] / w, q[7] / w);
        }
        for (auto& x : pv) x = 0;
        cudaMemcpyToSymbol(g_kprof, pv, sizeof(pv));
#endif
        fprintf(stderr, "[gicp knn] m=%lld levels=%d escalated=%d exact=%d bruteforce=%d tile-fallback=%d\n",
                (long long)m, L, h[2], h[0], h[1], h[3]);
        if (h[0] > 0) {
            int2 ex[16];
            const int ne = h[0] < 16 ? h[0] : 16;
            cudaMemcpyAsync(ex, exact, ne * sizeof(int2), cudaMemcpyDeviceToHost, s);
            cudaStreamSynchronize(s);
            for (int i = 0; i < ne; ++i) fprintf(stderr, "   exact id=%d level=%d\n", ex[i].x, ex[i].y);
        }
    }
    return check_cuda(cudaGetLastError(), "knn launch");
}

template <int KCAP>
int run_self(const gicp_index_s* idx, int k, float eps, int32_t* nbr, float* d2, float* cov, cudaStream_t s) {
    return run_queries<KCAP>(idx, nullptr, nullptr, idx->n, k, eps, nbr, d2, cov, s);
}

// the cell-sorted order of external queries (the order run_ext processes them in)
int query_order(const gicp_index_s* idx, const float* q, int64_t m, int* perm, cudaStream_t s) {
    Scratch keys_in, keys_out, vals_in, temp;
    int rc;
    if ((rc = keys_in.alloc(m * 8, s)) || (rc = keys_out.alloc(m * 8, s)) || (rc = vals_in.alloc(m * 4, s))) return rc;
    auto bits_for = [](int d) {
        int b = 0;
        while ((1 << b) < d) ++b;
        return b;
    };
    const Grid& g0 = idx->lv[0];
    const int bits = std::max(1, 3 * std::max(bits_for(g0.nx), std::max(bits_for(g0.ny), bits_for(g0.nz))));
    const unsigned long long empty = bits >= 64 ? kEmptyKey : (1ull << bits) - 1ull;
    k_query_keys<<<(unsigned)((m + 255) / 256), 256, 0, s>>>(q, m, g0, empty, (unsigned long long*)keys_in.p,
                                                              (int*)vals_in.p);
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, (unsigned long long*)keys_in.p, (unsigned long long*)keys_out.p,
                                    (int*)vals_in.p, perm, (int)m, 0, bits, s);
    if ((rc = temp.alloc(tb, s))) return rc;
    cub::DeviceRadixSort::SortPairs(temp.p, tb, (unsigned long long*)keys_in.p, (unsigned long long*)keys_out.p,
                                    (int*)vals_in.p, perm, (int)m, 0, bits, s);
    return check_cuda(cudaGetLastError(), "query order");
}

template <int KCAP>
int run_subset(const gicp_index_s* idx, const float* q, const int* ids, int64_t n_ids, int k, int32_t* nbr, float* d2,
               cudaStream_t s) {
    return run_queries<KCAP>(idx, q, ids, n_ids, k, 0.f, nbr, d2, nullptr, s);
}

template <int KCAP>
int run_ext(const gicp_index_s* idx, const float* q, int64_t m, int k, int32_t* nbr, float* d2, cudaStream_t s) {
    Scratch keys_in, keys_out, vals_in, perm, temp;
    int rc;
    if ((rc = keys_in.alloc(m * 8, s)) || (rc = keys_out.alloc(m * 8, s)) || (rc = vals_in.alloc(m * 4, s)) ||
        (rc = perm.alloc(m * 4, s)))
        return rc;
    // sort on the key bits in use (clamped voxel coordinates), not all 64
    auto bits_for = [](int d) {
        int b = 0;
        while ((1 << b) < d) ++b;
        return b;
    };
    const Grid& g0 = idx->lv[0];
    const int bits = std::max(1, 3 * std::max(bits_for(g0.nx), std::max(bits_for(g0.ny), bits_for(g0.nz))));
    const unsigned long long empty = bits >= 64 ? kEmptyKey : (1ull << bits) - 1ull;
    k_query_keys<<<(unsigned)((m + 255) / 256), 256, 0, s>>>(q, m, g0, empty, (unsigned long long*)keys_in.p,
                                                              (int*)vals_in.p);
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, (unsigned long long*)keys_in.p, (unsigned long long*)keys_out.p,
                                    (int*)vals_in.p, (int*)perm.p, (int)m, 0, bits, s);
    if ((rc = temp.alloc(tb, s))) return rc;
    cub::DeviceRadixSort::SortPairs(temp.p, tb, (unsigned long long*)keys_in.p, (unsigned long long*)keys_out.p,
                                    (int*)vals_in.p, (int*)perm.p, (int)m, 0, bits, s);
    return run_queries<KCAP>(idx, q, (int*)perm.p, m, k, 0.f, nbr, d2, nullptr, s);
}

}  // namespace

#define GICP_KCAP_DISPATCH(K, CALL)                      \
    switch ((K + 3) / 4) {                               \
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

int launch_knn_subset(const gicp_index_s* idx, const float* q, const int* ids, int64_t n_ids, int k, int32_t* nbr,
                      float* d2, cudaStream_t s) {
    GICP_KCAP_DISPATCH(k, (run_subset<KC>(idx, q, ids, n_ids, k, nbr, d2, s)));
}

int launch_query_order(const gicp_index_s* idx, const float* q, int64_t m, int* perm, cudaStream_t s) {
    return query_order(idx, q, m, perm, s);
}

}  // namespace gicp
