// knn_tile.cuh -- the tiled (cell-centric) fast path of the self kNN + covariance
// (included by knn.cu inside its anonymous namespace).
//
// Paper: "GPU-based nearest points search and covariance computation" (PAPER.md
// l.413, l.798); definition (R9): per query the k smallest keys (fp32 d2 in
// the fixed FMA order, ORIGINAL target index) over ALL targets.
//
// Work unit = one occupied level-1 voxel (a "tile": 2x2x2 level-0 voxels), one warp
// per tile. The warp stages into shared memory EVERY point of the 4x4x4 level-0 box
// around the tile (the tile's own points first, one bulk copy; then the 56 outer
// voxels nearest-first: faces, edges, corners) with TMA bulk copies
// (cp.async.bulk, one per non-empty voxel, completion on an mbarrier). Each lane then
// takes one of the tile's points as its query and scans the staged list in lockstep
// with the warp: every lane reads the same candidate (a shared-memory broadcast), no
// per-lane range bookkeeping. The top K+1 keys live in registers as 32-bit packed
// keys (bits(d2) with the low 9 bits replaced by the candidate's slot + 1), updated
// by comparator networks of single-instruction min/max (sortnet.cuh): the first 32
// candidates are sorted directly; later candidates below the current (K+1)-th key go
// to an 8-key register buffer, merged into the list when a lane's buffer fills.
//
// Exactness: the packed order equals the (d2, index) order except among keys whose
// d2 agree in their upper 23 bits. If no two adjacent keys of the K+1 list share
// them, the K smallest are exactly the first K in this order (every other candidate
// has a strictly larger d2). Otherwise (near-ties, exact ties) the query goes to the
// exact path. The query is final when the K-th d2 (an upper bound: low bits set) is
// below the squared distance from the query to the box boundary minus the grid's
// rounding slack (every point outside the box is farther); else it escalates to the
// pyramid path. Tiles with more than 511 staged points run the per-query level-0
// kernel instead.

constexpr int kTB = 128;        // queries (threads) per block: consecutive sorted positions
constexpr int kBlkTiles = 12;   // tiles a block may stage (sparser blocks: per-query kernel)
#ifndef GICP_TILE_BLKCAP
#define GICP_TILE_BLKCAP 1280  // (1536: 1.141 ms, 1280 + minBlocks 5: 1.109 ms, 1024: 1.12-1.13 ms on the C3 map)
#endif
constexpr int kBlkCap = GICP_TILE_BLKCAP;  // staged points per block (+ kTileCap of padding: unclamped reads)
constexpr int kSlotBits = 9;    // low key bits holding the candidate's slot + 1
constexpr unsigned kSlotMask = (1u << kSlotBits) - 1u;
constexpr int kTileCap = (int)kSlotMask;  // staged points per tile (slot + 1 fits the slot bits)
constexpr int kTileFirst = 32;  // candidates sorted directly before the buffered merges
constexpr int kTileBuf = 12;    // pending keys per lane (shared memory); merged once >= 8

// the 56 outer voxels of the box (offsets -1..2 per axis around the tile's 2x2x2
// block at 0..1), nearest-first: 24 face-, 24 edge-, 8 corner-adjacent
struct OuterCells {
    signed char d[56][3];
};
constexpr OuterCells make_outer_cells() {
    OuterCells o{};
    int n = 0;
    for (int cls = 1; cls <= 3; ++cls)
        for (int z = -1; z <= 2; ++z)
            for (int y = -1; y <= 2; ++y)
                for (int x = -1; x <= 2; ++x) {
                    const int out = (x < 0 || x > 1) + (y < 0 || y > 1) + (z < 0 || z > 1);
                    if (out != cls) continue;
                    o.d[n][0] = (signed char)x;
                    o.d[n][1] = (signed char)y;
                    o.d[n][2] = (signed char)z;
                    ++n;
                }
    return o;
}
__constant__ OuterCells c_outer = make_outer_cells();
// all 64 box cells, the tile's own 2x2x2 first (then nearest-first): external queries
struct BoxCells {
    signed char d[64][3];
};
constexpr BoxCells make_box_cells() {
    BoxCells b{};
    const OuterCells o = make_outer_cells();
    for (int i = 0; i < 8; ++i) {
        b.d[i][0] = (signed char)(i & 1);
        b.d[i][1] = (signed char)((i >> 1) & 1);
        b.d[i][2] = (signed char)(i >> 2);
    }
    for (int i = 0; i < 56; ++i)
        for (int a = 0; a < 3; ++a) b.d[8 + i][a] = o.d[i][a];
    return b;
}
__constant__ BoxCells c_box = make_box_cells();

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
// TMA bulk copy global -> shared (16-B aligned, multiple of 16 bytes), completing on bar
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ unsigned pack_key(float d2, int slot) {
    return (__float_as_uint(d2) & ~kSlotMask) | (unsigned)(slot + 1);
}

// merge the lane's pending keys (buf[0..nb) of its shared-memory column) into the
// sorted (K+1)-list
template <int NL>
__device__ __forceinline__ void tile_merge(unsigned (&T)[NL], const unsigned* __restrict__ col, int nb) {
    constexpr net::Net sb = net::make_sort_net<kTileBuf, kTileBuf>();
    constexpr net::Net mg = net::make_merge_net<NL, kTileBuf, NL>();
    unsigned b[kTileBuf];
#pragma unroll
    for (int i = 0; i < kTileBuf; ++i) b[i] = i < nb ? col[i * kTB] : 0xffffffffu;
    GICP_APPLY_NET(b, sb);
    unsigned w[NL + kTileBuf];
#pragma unroll
    for (int i = 0; i < NL; ++i) w[i] = T[i];
#pragma unroll
    for (int i = 0; i < kTileBuf; ++i) w[NL + i] = b[sb.out[i]];
    GICP_APPLY_NET(w, mg);
#pragma unroll
    for (int i = 0; i < NL; ++i) T[i] = w[mg.out[i]];
}

// exact (d2, original index) order of two staged candidates for query q
__device__ __forceinline__ bool exact_less(const float4& q, const float4& a, const float4& b) {
    const float da = dist2(q.x, q.y, q.z, a.x, a.y, a.z), db = dist2(q.x, q.y, q.z, b.x, b.y, b.z);
    return da < db || (da == db && __float_as_int(a.w) < __float_as_int(b.w));
}

#ifndef GICP_TILE_MINB
#define GICP_TILE_MINB 5
#endif
// ROWS: each lane scans only the 27 voxels around its own (nine x-rows of three
// voxels of the box, staged in (z, y, x) order so every row is contiguous) and the
// stop rule uses that cube; the block's lanes are regrouped by the parity of their
// voxel (the same relative rows), so a warp's lanes step through the same rows.
// EXT: external queries (gicp_knn): the block's 128 queries are consecutive in their
// cell-sorted order (perm); a "tile" is each distinct level-1 voxel of their (clamped)
// cells, its whole 4x4x4 box probed and staged, the tile's own 2x2x2 first; rows go
// to the queries' original indices, no covariance. Non-finite queries: per-query path.
template <int K, bool ROWS, bool EXT = false>
__global__ void __launch_bounds__(kTB, K <= 20 ? GICP_TILE_MINB : 4) k_knn_tile(const float4* __restrict__ pts, Grid g0,
                                                  const int* __restrict__ tiles, const int* __restrict__ tile_of,
                                                  int64_t n, float eps, int32_t* __restrict__ nbr,
                                                  float* __restrict__ d2out, float* __restrict__ cov,
                                                  int* __restrict__ esc_count, int* __restrict__ esc_list,
                                                  int* __restrict__ exact_count, int2* __restrict__ exact_list,
                                                  int* __restrict__ fb_count, int* __restrict__ fb_list,
                                                  const float* __restrict__ qext = nullptr,
                                                  const int* __restrict__ perm = nullptr) {
    static_assert(!(ROWS && EXT), "external queries use the box scan");
    constexpr int NL = K + 1;
    __shared__ __align__(128) float4 cand[kBlkCap + kTileCap + 4];
    __shared__ unsigned buf[kTileBuf][kTB];
    constexpr int NR = (ROWS || EXT) ? 64 : 57;  // staged ranges per tile
    __shared__ int2 rng[kBlkTiles][NR];
    __shared__ int cell_off[ROWS ? kBlkTiles : 1][65];  // ROWS: box cell starts in cand, then the end
    __shared__ int s_order[ROWS ? kTB : 1], s_pc[8];
    __shared__ unsigned long long s_l1[EXT ? kTB : 1];
    __shared__ int s_run[EXT ? kTB : 1], s_wst[kTB / 32];
    __shared__ int t_off[kBlkTiles], t_cnt[kBlkTiles], t_start[kBlkTiles], t_base[kBlkTiles][3];
    __shared__ __align__(8) unsigned long long bar;
    __shared__ int s_ta, s_nt, s_ok;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t q0 = (int64_t)blockIdx.x * kTB, q = q0 + tid;
    const bool act = q < n;  // EXT: n = the number of queries
    // EXT: this lane's query
    int qid = (int)q;
    float ex = 0.f, ey = 0.f, ez = 0.f;
    bool efin = false;
    if (EXT && act) {
        qid = __ldg(perm + q);
        ex = __ldg(qext + 3 * (int64_t)qid);
        ey = __ldg(qext + 3 * (int64_t)qid + 1);
        ez = __ldg(qext + 3 * (int64_t)qid + 2);
        efin = isfinite(ex) && isfinite(ey) && isfinite(ez);
    }
    if (tid == 0) mbar_init(&bar, 1);
    if constexpr (EXT) {
        // runs of equal level-1 voxels (clamped cells, the sort's key) = the tiles
        unsigned long long k1 = ~0ull;
        int cx = 0, cy = 0, cz = 0;
        if (efin) {
            cx = min(max(cell_coord(ex, g0.ox, g0.inv_cell), 0), g0.nx - 1);
            cy = min(max(cell_coord(ey, g0.oy, g0.inv_cell), 0), g0.ny - 1);
            cz = min(max(cell_coord(ez, g0.oz, g0.inv_cell), 0), g0.nz - 1);
            k1 = cell_key(cx >> 1, cy >> 1, cz >> 1);
        }
        s_l1[tid] = k1;
        __syncthreads();
        const bool st = efin && (tid == 0 || s_l1[tid - 1] != k1);
        const unsigned bm = __ballot_sync(0xffffffffu, st);
        if (lane == 0) s_wst[warp] = __popc(bm);
        __syncthreads();
        int before = 0, tot = 0;
        for (int w = 0; w < kTB / 32; ++w) {
            if (w < warp) before += s_wst[w];
            tot += s_wst[w];
        }
        const int r = before + __popc(bm & ((2u << lane) - 1u)) - 1;  // this lane's run
        if (st && r < kBlkTiles) {
            t_base[r][0] = cx & ~1;
            t_base[r][1] = cy & ~1;
            t_base[r][2] = cz & ~1;
        }
        s_run[tid] = r;
        if (tid == 0) {
            s_ta = 0;
            s_nt = tot;
        }
    } else if (tid == 0) {
        const int ta = __ldg(tile_of + q0), tb = __ldg(tile_of + min(q0 + kTB, n) - 1);
        s_ta = ta;
        s_nt = tb - ta + 1;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    const int ta = s_ta, nt = s_nt;
    auto fallback_all = [&]() { push_warp(fb_count, fb_list, EXT ? (act && efin) : act, qid); };
    if (EXT) push_warp(fb_count, fb_list, act && !efin, qid);  // non-finite: the per-query path
    if (nt > kBlkTiles) {  // sparse region: many tiny tiles
        fallback_all();
        return;
    }
    // (1) per tile (warp w: tiles w, w + 4): the ranges of its box
    for (int lt = warp; lt < nt; lt += kTB / 32) {
        int s1 = 0, e1 = 0, bx, by, bz;
        if constexpr (EXT) {
            bx = t_base[lt][0];
            by = t_base[lt][1];
            bz = t_base[lt][2];
        } else {
            const int t = ta + lt;
            s1 = __ldg(tiles + t);
            e1 = __ldg(tiles + t + 1);
            const float4 f0 = __ldg(pts + s1);
            bx = cell_coord(f0.x, g0.ox, g0.inv_cell) & ~1;
            by = cell_coord(f0.y, g0.oy, g0.inv_cell) & ~1;
            bz = cell_coord(f0.z, g0.oz, g0.inv_cell) & ~1;
        }
        int2 ra, rb = make_int2(0, 0);
        if constexpr (EXT) {  // all 64 box cells, the tile's own first
            const signed char* d = c_box.d[lane];
            const signed char* e = c_box.d[lane + 32];
            ra = cell_lookup(g0, bx + d[0], by + d[1], bz + d[2]);
            rb = cell_lookup(g0, bx + e[0], by + e[1], bz + e[2]);
        } else if constexpr (ROWS) {  // box cell ci = (z * 4 + y) * 4 + x, offsets -1..2 per axis
            ra = cell_lookup(g0, bx - 1 + (lane & 3), by - 1 + ((lane >> 2) & 3), bz - 1 + (lane >> 4));
            const int c2 = lane + 32;
            rb = cell_lookup(g0, bx - 1 + (c2 & 3), by - 1 + ((c2 >> 2) & 3), bz - 1 + (c2 >> 4));
        } else {
            const signed char* d = c_outer.d[lane];
            ra = cell_lookup(g0, bx + d[0], by + d[1], bz + d[2]);
            if (lane < 24) {
                const signed char* e = c_outer.d[lane + 32];
                rb = cell_lookup(g0, bx + e[0], by + e[1], bz + e[2]);
            }
        }
        const int ca = max(ra.y - ra.x, 0), cb = max(rb.y - rb.x, 0);
        if constexpr (ROWS || EXT) {
            rng[lt][lane] = make_int2(ra.x, ca);
            rng[lt][32 + lane] = make_int2(rb.x, cb);
        } else {
            rng[lt][1 + lane] = make_int2(ra.x, ca);
            if (lane < 24) rng[lt][33 + lane] = make_int2(rb.x, cb);
        }
        const int tot = __reduce_add_sync(0xffffffffu, ca + cb);
        if (lane == 0) {
            if (!ROWS && !EXT) rng[lt][0] = make_int2(s1, e1 - s1);
            t_cnt[lt] = ((ROWS || EXT) ? 0 : e1 - s1) + tot;
            t_start[lt] = s1;
            t_base[lt][0] = bx;
            t_base[lt][1] = by;
            t_base[lt][2] = bz;
        }
    }
    __syncthreads();
    if (tid == 0) {
        int o = 0, ok = 1;
        for (int lt = 0; lt < nt; ++lt) {
            t_off[lt] = o;
            o += t_cnt[lt];
            ok &= t_cnt[lt] <= kTileCap;
        }
        ok &= o <= kBlkCap;
        s_ok = ok;
        if (ok) mbar_arrive_expect_tx(&bar, (unsigned)o * 16u);
    }
    __syncthreads();
    if (!s_ok) {  // a tile too dense to stage
        fallback_all();
        return;
    }
    // (2) one TMA bulk copy per non-empty range, completion on the block's barrier
    for (int lt = warp; lt < nt; lt += kTB / 32) {
        const int2 a = rng[lt][lane];
        const int2 b = lane + 32 < NR ? rng[lt][lane + 32] : make_int2(0, 0);
        int ia = a.y, ib = b.y;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int va = __shfl_up_sync(0xffffffffu, ia, o), vb = __shfl_up_sync(0xffffffffu, ib, o);
            if (lane >= o) {
                ia += va;
                ib += vb;
            }
        }
        const int tot_a = __shfl_sync(0xffffffffu, ia, 31);
        const int oa = t_off[lt] + ia - a.y, ob = t_off[lt] + tot_a + ib - b.y;
        if (a.y > 0) bulk_g2s(cand + oa, pts + a.x, (unsigned)a.y * 16u, &bar);
        if (b.y > 0) bulk_g2s(cand + ob, pts + b.x, (unsigned)b.y * 16u, &bar);
        if (ROWS) {
            cell_off[lt][lane] = oa;
            cell_off[lt][32 + lane] = ob;
            if (lane == 31) cell_off[lt][64] = ob + b.y;
        }
    }
    if (ROWS) {
        // regroup the block's queries by the parity of their voxel (which of the
        // tile's 2x2x2 voxels): lanes of one group scan the same relative rows
        if (tid < 8) s_pc[tid] = 0;
        __syncthreads();
        int par = 0, rk = 0;
        if (act) {
            const float4 pq = __ldg(pts + q);
            par = (cell_coord(pq.x, g0.ox, g0.inv_cell) & 1) | ((cell_coord(pq.y, g0.oy, g0.inv_cell) & 1) << 1) |
                  ((cell_coord(pq.z, g0.oz, g0.inv_cell) & 1) << 2);
            rk = atomicAdd(&s_pc[par], 1);
        }
        __syncthreads();
        if (act) {
            int b0 = 0;
            for (int i = 0; i < par; ++i) b0 += s_pc[i];
            s_order[b0 + rk] = tid;
        }
        __syncthreads();
    }
    mbar_wait(&bar, 0);
    // (3) per lane: its query and its tile's staged box
    int lt = 0, base = 0, C = 0;
    float4 qp = make_float4(0.f, 0.f, 0.f, 0.f);
    const int nq = (int)min((int64_t)kTB, n - q0);
    const int me = ROWS ? (tid < nq ? s_order[tid] : tid) : tid;  // the lane's query (block-relative)
    const int64_t qq = EXT ? (int64_t)qid : q0 + me;               // its id in the lists / rows
    const bool on = ROWS ? tid < nq : (EXT ? act && efin : act);
    if (on) {
        lt = EXT ? s_run[tid] : __ldg(tile_of + qq) - ta;
        base = t_off[lt];
        C = t_cnt[lt];
        qp = EXT ? make_float4(ex, ey, ez, 0.f) : (ROWS ? __ldg(pts + qq) : cand[base + (int)(qq - t_start[lt])]);
    }
    unsigned T[NL];
    unsigned* col = &buf[0][tid];
    int nb = 0;
    if constexpr (ROWS) {
#pragma unroll
        for (int i = 0; i < NL; ++i) T[i] = 0xffffffffu;
        unsigned thr = 0xffffffffu;
        int ix = 0, iy = 0, iz = 0;
        if (on) {
            ix = cell_coord(qp.x, g0.ox, g0.inv_cell) - t_base[lt][0] + 1;
            iy = cell_coord(qp.y, g0.oy, g0.inv_cell) - t_base[lt][1] + 1;
            iz = cell_coord(qp.z, g0.oz, g0.inv_cell) - t_base[lt][2] + 1;
        }
        // the nine rows (dz, dy), nearest first; each covers x = ix-1 .. ix+1
        constexpr signed char kRow[9][2] = {{0, 0}, {0, -1}, {0, 1}, {-1, 0}, {1, 0},
                                            {-1, -1}, {-1, 1}, {1, -1}, {1, 1}};
#pragma unroll 1
        for (int r = 0; r < 9; ++r) {
            int a = 0, len = 0;
            if (on) {
                const int ci = ((iz + kRow[r][0]) * 4 + (iy + kRow[r][1])) * 4 + ix - 1;
                a = cell_off[lt][ci];
                len = cell_off[lt][ci + 3] - a;
            }
            const int rel = a - base;  // slot of the row's first point within the tile
            const int lmax = __reduce_max_sync(0xffffffffu, len);
            for (int c = 0; c < lmax; c += 4) {
                unsigned kk[4];
                bool ps[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int cc = c + u;
                    const float4 p = cand[a + cc];  // past len: padding or other points (masked below)
                    const float dd = dist2(qp.x, qp.y, qp.z, p.x, p.y, p.z);
                    ps[u] = cc < len && __float_as_uint(dd) <= thr;
                    kk[u] = pack_key(dd, rel + cc);
                }
                if (__any_sync(0xffffffffu, ps[0] | ps[1] | ps[2] | ps[3])) {
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        if (ps[u]) col[(nb++) * kTB] = kk[u];
                    if (__any_sync(0xffffffffu, nb >= kTileBuf - 4)) {
                        tile_merge<NL>(T, col, nb);
                        nb = 0;
                        thr = T[NL - 1] | kSlotMask;
                    }
                }
            }
        }
    } else {
        // (K = 32: the list has 33 places and the first sort 32 keys; the last place
        // starts empty)
        constexpr int NF = NL < kTileFirst ? NL : kTileFirst;
        constexpr net::Net sn = net::make_sort_net<kTileFirst, NF>();
        unsigned v[kTileFirst];
#pragma unroll
        for (int i = 0; i < kTileFirst; ++i) {
            v[i] = 0xffffffffu;
            if (i < C) {
                const float4 p = cand[base + i];
                v[i] = pack_key(dist2(qp.x, qp.y, qp.z, p.x, p.y, p.z), i);
            }
        }
        GICP_APPLY_NET(v, sn);
#pragma unroll
        for (int i = 0; i < NL; ++i) T[i] = i < NF ? v[sn.out[i]] : 0xffffffffu;
    unsigned thr = T[NL - 1] | kSlotMask;
    const int cmax = __reduce_max_sync(0xffffffffu, C);
    for (int c = kTileFirst; c < cmax; c += 4) {
        unsigned kk[4];
        bool ps[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int cc = c + u;
            const float4 p = cand[base + cc];  // past C: padding or the next tile (masked below)
            const float dd = dist2(qp.x, qp.y, qp.z, p.x, p.y, p.z);
            ps[u] = cc < C && __float_as_uint(dd) <= thr;
            kk[u] = pack_key(dd, cc);
        }
        if (__any_sync(0xffffffffu, ps[0] | ps[1] | ps[2] | ps[3])) {
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (ps[u]) col[(nb++) * kTB] = kk[u];
            if (__any_sync(0xffffffffu, nb >= kTileBuf - 4)) {
                tile_merge<NL>(T, col, nb);
                nb = 0;
                thr = T[NL - 1] | kSlotMask;
            }
        }
    }
    }  // ROWS
    if (__any_sync(0xffffffffu, nb > 0)) tile_merge<NL>(T, col, nb);
    // (4) order certainty. (a) Boundary near-tie: the K-th and (K+1)-th keys share
    // their d2 prefix U, so candidates with prefix U (some maybe past the list) decide
    // the last places: rank them by the exact key (d2 bits, original index) in a
    // rescan and rewrite list places lo..K-1 (rare: a few per mille of the queries).
    int st = 0;  // 0 emit, 1 escalate, 2 exact path
    bool amb_b = on && (T[K - 1] >> kSlotBits) == (T[K] >> kSlotBits) && T[K - 1] != 0xffffffffu;
    if (__any_sync(0xffffffffu, amb_b)) {
        constexpr int KB = 4;  // places resolved in-kernel (more: the exact path)
        const unsigned U = T[K - 1] >> kSlotBits;
        int lo = 0;
#pragma unroll
        for (int r = 0; r < K; ++r) lo += (T[r] >> kSlotBits) < U ? 1 : 0;
        const int need = K - lo;
        unsigned long long ek[KB];
        int es[KB];
#pragma unroll
        for (int i = 0; i < KB; ++i) {
            ek[i] = ~0ull;
            es[i] = 0;
        }
        const int cm = __reduce_max_sync(0xffffffffu, amb_b ? C : 0);
        for (int c = 0; c < cm; ++c) {
            const float4 p = cand[base + c];
            const float dd = dist2(qp.x, qp.y, qp.z, p.x, p.y, p.z);
            const bool take = amb_b && c < C && (__float_as_uint(dd) >> kSlotBits) == U;
            const unsigned long long key =
                take ? (((unsigned long long)__float_as_uint(dd) << 32) | (unsigned)__float_as_int(p.w)) : ~0ull;
            // sorted insertion into the KB-list (no-op for ~0)
            bool below = key < ek[KB - 1];
#pragma unroll
            for (int r = KB - 1; r > 0; --r) {
                const bool sh = below && key < ek[r - 1];
                const bool put = below && !sh;
                const unsigned long long nk = sh ? ek[r - 1] : (put ? key : ek[r]);
                const int ns = sh ? es[r - 1] : (put ? c : es[r]);
                ek[r] = nk;
                es[r] = ns;
                below = sh;
            }
            if (below) {
                ek[0] = key;
                es[0] = c;
            }
        }
        if (amb_b && need >= 1 && need <= KB) {
#pragma unroll
            for (int r = 0; r < K; ++r)
#pragma unroll
                for (int j2 = 0; j2 < KB; ++j2)
                    if (j2 < need && r == lo + j2) T[r] = (U << kSlotBits) | (unsigned)(es[j2] + 1);
            amb_b = false;
        }
    }
    // (b) near-equal neighbours inside the list: their packed order must be the exact
    // one; two passes of exact compare-exchange fix groups of up to three, anything
    // left goes to the exact path
    bool amb_in = false;
    if (on) {
#pragma unroll
        for (int r = 0; r < K - 1; ++r) amb_in |= (T[r] >> kSlotBits) == (T[r + 1] >> kSlotBits);
    }
    if (__any_sync(0xffffffffu, amb_in)) {
        bool bad = false;
        if (amb_in) {
            for (int pass = 0; pass < 3; ++pass) {
                bad = false;
#pragma unroll
                for (int r = 0; r < K - 1; ++r)
                    if ((T[r] >> kSlotBits) == (T[r + 1] >> kSlotBits) &&
                        !exact_less(qp, cand[base + (int)(T[r] & kSlotMask) - 1],
                                    cand[base + (int)(T[r + 1] & kSlotMask) - 1])) {
                        if (pass < 2) {
                            const unsigned t = T[r];
                            T[r] = T[r + 1];
                            T[r + 1] = t;
                        }
                        bad = true;
                    }
                if (!bad) break;
            }
        }
        amb_in = bad;
    }
    if (on) {
        const int bx = t_base[lt][0], by = t_base[lt][1], bz = t_base[lt][2];
        const float s = g0.cell;
        const float kth = __uint_as_float(T[K - 1] | kSlotMask);  // >= the K-th d2
        const QGeom G = make_geom(g0, qp.x, qp.y, qp.z);
        float m;
        if (ROWS) {  // the 27-voxel cube around the query's voxel
            m = cube_margin(G, s, g0.slack, 1);
        } else {     // the tile's box
            const float mx = fminf(G.fx + (float)(G.cx - bx + 1) * s, (float)(bx + 3 - G.cx) * s - G.fx);
            const float my = fminf(G.fy + (float)(G.cy - by + 1) * s, (float)(by + 3 - G.cy) * s - G.fy);
            const float mz = fminf(G.fz + (float)(G.cz - bz + 1) * s, (float)(bz + 3 - G.cz) * s - G.fz);
            m = fminf(mx, fminf(my, mz)) - g0.slack;
        }
        const bool full = T[K - 1] != 0xffffffffu;
        const bool fin = full && m > 0.0f && kth < m * m * kRel;
        st = !fin ? 1 : ((amb_in || amb_b) ? 2 : 0);
    }
    push_warp(esc_count, esc_list, on && st == 1, (int)qq);
    push_warp2(exact_count, exact_list, on && st == 2, make_int2((int)qq, 0));
    if (!on || st != 0) return;
    // (5) emit: original indices, exact d2, covariance of the K neighbours
    const int64_t row = EXT ? (int64_t)qid : (int64_t)__float_as_int(qp.w);
    const float4 p0 = cand[base + (int)(T[0] & kSlotMask) - 1];
    float sx = 0.f, sy = 0.f, sz = 0.f;
    // rows written 4 (K % 4 == 0), 2 or 1 values at a time as they are formed
    constexpr int VW = (K % 4 == 0) ? 4 : ((K % 2 == 0) ? 2 : 1);
#pragma unroll
    for (int r0 = 0; r0 < K; r0 += VW) {
        int ids[VW];
        float dd[VW];
#pragma unroll
        for (int u = 0; u < VW; ++u) {
            const float4 p = cand[base + (int)(T[r0 + u] & kSlotMask) - 1];
            ids[u] = __float_as_int(p.w);
            dd[u] = dist2(qp.x, qp.y, qp.z, p.x, p.y, p.z);
            sx += p.x - p0.x;
            sy += p.y - p0.y;
            sz += p.z - p0.z;
        }
        if (VW == 4) {
            if (nbr) *reinterpret_cast<int4*>(nbr + row * K + r0) = make_int4(ids[0], ids[1 % VW], ids[2 % VW], ids[3 % VW]);
            if (d2out)
                *reinterpret_cast<float4*>(d2out + row * K + r0) = make_float4(dd[0], dd[1 % VW], dd[2 % VW], dd[3 % VW]);
        } else if (VW == 2) {
            if (nbr) *reinterpret_cast<int2*>(nbr + row * K + r0) = make_int2(ids[0], ids[1 % VW]);
            if (d2out) *reinterpret_cast<float2*>(d2out + row * K + r0) = make_float2(dd[0], dd[1 % VW]);
        } else {
            if (nbr) nbr[row * K + r0] = ids[0];
            if (d2out) d2out[row * K + r0] = dd[0];
        }
    }
    if (!cov) return;
    const float invk = 1.0f / (float)K;
    const float mxm = sx * invk, mym = sy * invk, mzm = sz * invk;
    float c00 = 0.f, c01 = 0.f, c02 = 0.f, c11 = 0.f, c12 = 0.f, c22 = 0.f;
#pragma unroll
    for (int r = 0; r < K; ++r) {
        const float4 p = cand[base + (int)(T[r] & kSlotMask) - 1];
        const float x = (p.x - p0.x) - mxm, y = (p.y - p0.y) - mym, z = (p.z - p0.z) - mzm;
        c00 = fmaf(x, x, c00);
        c01 = fmaf(x, y, c01);
        c02 = fmaf(x, z, c02);
        c11 = fmaf(y, y, c11);
        c12 = fmaf(y, z, c12);
        c22 = fmaf(z, z, c22);
    }
    float cc[6];
    plane_cov(c00 * invk, c01 * invk, c02 * invk, c11 * invk, c12 * invk, c22 * invk, eps, cc);
    store_cov(cov, row, cc);
}
