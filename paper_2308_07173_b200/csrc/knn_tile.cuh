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
// keys (bits(d2) with the low 8 bits replaced by the candidate's slot + 1), updated
// by comparator networks of single-instruction min/max (sortnet.cuh): the first 32
// candidates are sorted directly; later candidates below the current (K+1)-th key go
// to an 8-key register buffer, merged into the list when a lane's buffer fills.
//
// Exactness: the packed order equals the (d2, index) order except among keys whose
// d2 agree in their upper 24 bits. If no two adjacent keys of the K+1 list share
// them, the K smallest are exactly the first K in this order (every other candidate
// has a strictly larger d2). Otherwise (near-ties, exact ties) the query goes to the
// exact path. The query is final when the K-th d2 (an upper bound: low bits set) is
// below the squared distance from the query to the box boundary minus the grid's
// rounding slack (every point outside the box is farther); else it escalates to the
// pyramid path. Tiles with more than 255 staged points run the per-query level-0
// kernel instead.

constexpr int kTileWarps = 4;
constexpr int kTileCap = 255;  // staged points per tile (slot + 1 fits 8 bits)
constexpr int kTileFirst = 32; // candidates sorted directly before the buffered merges
constexpr int kTileBuf = 8;    // pending keys per lane

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
    return (__float_as_uint(d2) & 0xffffff00u) | (unsigned)(slot + 1);
}

// merge the 8-key buffer into the sorted (K+1)-list; buffer reset to empty
template <int NL>
__device__ __forceinline__ void tile_merge(unsigned (&T)[NL], unsigned (&B)[kTileBuf]) {
    constexpr net::Net s8 = net::make_sort_net<kTileBuf, kTileBuf>();
    unsigned w[NL + kTileBuf];
#pragma unroll
    for (int i = 0; i < kTileBuf; ++i) w[i] = B[i];
    {
        unsigned b8[kTileBuf];
#pragma unroll
        for (int i = 0; i < kTileBuf; ++i) b8[i] = B[i];
        GICP_APPLY_NET(b8, s8);
#pragma unroll
        for (int i = 0; i < kTileBuf; ++i) w[NL + i] = b8[s8.out[i]];
    }
#pragma unroll
    for (int i = 0; i < NL; ++i) w[i] = T[i];
    constexpr net::Net mg = net::make_merge_net<NL, kTileBuf, NL>();
    GICP_APPLY_NET(w, mg);
#pragma unroll
    for (int i = 0; i < NL; ++i) T[i] = w[mg.out[i]];
#pragma unroll
    for (int i = 0; i < kTileBuf; ++i) B[i] = 0xffffffffu;
}

template <int K>
__global__ void __launch_bounds__(kTileWarps * 32) k_knn_tile(const float4* __restrict__ pts, Grid g0,
                                                              const int* __restrict__ tiles, int64_t ntiles, float eps,
                                                              int32_t* __restrict__ nbr, float* __restrict__ d2out,
                                                              float* __restrict__ cov, int* __restrict__ esc_count,
                                                              int* __restrict__ esc_list, int* __restrict__ exact_count,
                                                              int2* __restrict__ exact_list,
                                                              int* __restrict__ fb_count, int* __restrict__ fb_list) {
    constexpr int NL = K + 1;
    __shared__ __align__(128) float4 s_cand[kTileWarps][kTileCap + 1];
    __shared__ __align__(8) unsigned long long s_bar[kTileWarps];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float4* cand = s_cand[warp];
    unsigned long long* bar = &s_bar[warp];
    if (lane == 0) mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    unsigned phase = 0;
    const float s = g0.cell, slack = g0.slack;
    for (int64_t t = (int64_t)blockIdx.x * kTileWarps + warp; t < ntiles; t += (int64_t)gridDim.x * kTileWarps) {
        const int s1 = __ldg(tiles + t), e1 = __ldg(tiles + t + 1);
        const int Q = e1 - s1;
        // the tile's level-0 base coordinates (even): the level-1 voxel of its first point
        const float4 f0 = __ldg(pts + s1);
        const int bx = cell_coord(f0.x, g0.ox, g0.inv_cell) & ~1;
        const int by = cell_coord(f0.y, g0.oy, g0.inv_cell) & ~1;
        const int bz = cell_coord(f0.z, g0.oz, g0.inv_cell) & ~1;
        // the 56 outer voxels: lane takes outer cells lane and lane + 32
        int2 ra = make_int2(0, 0), rb = make_int2(0, 0);
        {
            const signed char* d = c_outer.d[lane];
            ra = cell_lookup(g0, bx + d[0], by + d[1], bz + d[2]);
            if (lane < 24) {
                const signed char* e = c_outer.d[lane + 32];
                rb = cell_lookup(g0, bx + e[0], by + e[1], bz + e[2]);
            }
        }
        const int ca = max(ra.y - ra.x, 0), cb = max(rb.y - rb.x, 0);
        // offsets: inner block [0, Q), then the outer voxels in table order
        int ia = ca, ib = cb;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int va = __shfl_up_sync(0xffffffffu, ia, o), vb = __shfl_up_sync(0xffffffffu, ib, o);
            if (lane >= o) {
                ia += va;
                ib += vb;
            }
        }
        const int tot_a = __shfl_sync(0xffffffffu, ia, 31), tot_b = __shfl_sync(0xffffffffu, ib, 31);
        const int oa = Q + ia - ca, ob = Q + tot_a + ib - cb;
        const int C = Q + tot_a + tot_b;
        if (C > kTileCap) {  // dense tile: the per-query level-0 kernel
            for (int q0 = 0; q0 < Q; q0 += 32) {
                const bool a = q0 + lane < Q;
                push_warp(fb_count, fb_list, a, s1 + q0 + lane);
            }
            continue;
        }
        // stage the box: one bulk copy per non-empty range, completion on the barrier
        if (lane == 0) {
            mbar_arrive_expect_tx(bar, (unsigned)C * 16u);
            bulk_g2s(cand, pts + s1, (unsigned)Q * 16u, bar);
        }
        __syncwarp();
        if (ca > 0) bulk_g2s(cand + oa, pts + ra.x, (unsigned)ca * 16u, bar);
        if (cb > 0) bulk_g2s(cand + ob, pts + rb.x, (unsigned)cb * 16u, bar);
        mbar_wait(bar, phase);
        phase ^= 1u;

        for (int q0 = 0; q0 < Q; q0 += 32) {
            const int qi = q0 + lane;
            const bool act = qi < Q;
            const float4 qp = cand[act ? qi : q0];
            // (1) the first kTileFirst candidates, sorted directly
            unsigned T[NL];
            {
                constexpr net::Net sn = net::make_sort_net<kTileFirst, NL>();
                unsigned v[kTileFirst];
#pragma unroll
                for (int i = 0; i < kTileFirst; ++i) {
                    v[i] = 0xffffffffu;
                    if (i < C) {
                        const float4 p = cand[i];
                        v[i] = pack_key(dist2(qp.x, qp.y, qp.z, p.x, p.y, p.z), i);
                    }
                }
                GICP_APPLY_NET(v, sn);
#pragma unroll
                for (int i = 0; i < NL; ++i) T[i] = v[sn.out[i]];
            }
            // (2) the rest: keys below the current (K+1)-th go through the buffer
            unsigned B[kTileBuf];
#pragma unroll
            for (int i = 0; i < kTileBuf; ++i) B[i] = 0xffffffffu;
            int nb = 0;
            unsigned thr = T[NL - 1];
            for (int c = kTileFirst; c < C; ++c) {
                const float4 p = cand[c];
                const unsigned key = pack_key(dist2(qp.x, qp.y, qp.z, p.x, p.y, p.z), c);
                const bool pass = act && key < thr;
                if (__any_sync(0xffffffffu, pass)) {
#pragma unroll
                    for (int i = kTileBuf - 1; i > 0; --i) B[i] = pass ? B[i - 1] : B[i];
                    B[0] = pass ? key : B[0];
                    nb += pass ? 1 : 0;
                    if (__any_sync(0xffffffffu, nb == kTileBuf)) {
                        tile_merge<NL>(T, B);
                        nb = 0;
                        thr = T[NL - 1];
                    }
                }
            }
            if (__any_sync(0xffffffffu, nb > 0)) tile_merge<NL>(T, B);
            // (3) decisions: enough candidates, stop rule on the box, near-ties
            int st = 0;  // 0 emit, 1 escalate, 2 exact path
            if (act) {
                bool amb = false;
#pragma unroll
                for (int r = 0; r < K; ++r) amb |= (T[r] >> 8) == (T[r + 1] >> 8);
                const float kth = __uint_as_float(T[K - 1] | 0xffu);  // >= the K-th d2
                const QGeom G = make_geom(g0, qp.x, qp.y, qp.z);
                const float mx = fminf(G.fx + (float)(G.cx - bx + 1) * s, (float)(bx + 3 - G.cx) * s - G.fx);
                const float my = fminf(G.fy + (float)(G.cy - by + 1) * s, (float)(by + 3 - G.cy) * s - G.fy);
                const float mz = fminf(G.fz + (float)(G.cz - bz + 1) * s, (float)(bz + 3 - G.cz) * s - G.fz);
                const float m = fminf(mx, fminf(my, mz)) - slack;
                const bool full = T[K - 1] != 0xffffffffu;
                const bool fin = full && m > 0.0f && kth < m * m * kRel;
                st = !fin ? 1 : (amb ? 2 : 0);
            }
            push_warp(esc_count, esc_list, act && st == 1, s1 + qi);
            push_warp2(exact_count, exact_list, act && st == 2, make_int2(s1 + qi, 0));
            if (!act || st != 0) continue;
            // (4) emit: original indices, exact d2, covariance of the K neighbours
            const int64_t row = __float_as_int(qp.w);
            const float4 p0 = cand[(T[0] & 0xffu) - 1];
            float sx = 0.f, sy = 0.f, sz = 0.f;
            // rows written 4 (K % 4 == 0), 2 or 1 values at a time as they are formed
            constexpr int VW = (K % 4 == 0) ? 4 : ((K % 2 == 0) ? 2 : 1);
#pragma unroll
            for (int r0 = 0; r0 < K; r0 += VW) {
                int ids[VW];
                float dd[VW];
#pragma unroll
                for (int u = 0; u < VW; ++u) {
                    const float4 p = cand[(T[r0 + u] & 0xffu) - 1];
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
            if (!cov) continue;
            const float invk = 1.0f / (float)K;
            const float mxm = sx * invk, mym = sy * invk, mzm = sz * invk;
            float c00 = 0.f, c01 = 0.f, c02 = 0.f, c11 = 0.f, c12 = 0.f, c22 = 0.f;
#pragma unroll
            for (int r = 0; r < K; ++r) {
                const float4 p = cand[(T[r] & 0xffu) - 1];
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
        // the next tile's bulk copies overwrite the buffer: order this warp's reads
        // (generic proxy) before them (async proxy)
        __syncwarp();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
}
