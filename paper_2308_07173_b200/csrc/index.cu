// index.cu -- gicp_build_index: a uniform voxel grid built by radix sort on cell
// keys, extended to a pyramid of voxel levels that share one sorted array.
//
// Paper: the structure behind "GPU-based nearest points search" (PAPER.md l.413,
// "GPU-hash data structure" l.477); north star: "a uniform voxel grid built by
// radix sort on cell keys". Steps:
//   1. k_bbox        finiteness check + bounding box (warp reduce, ordered-int atomics)
//   2. k_keys        key_i = Morton(floor(fl32(fl32(x - o) * inv)) per axis)
//   3. CUB radix sort of (key, i) on the 3 x ceil(log2 dim) key bits in use
//   4. k_level_count occupied voxels of every level (key >> 3l changes)
//   5. k_cells / k_cell_ends   per level: run heads insert {key, start}, run tails
//                    write end (O(1) per point for any occupancy)
//   6. k_scatter     sorted float4 (x, y, z, orig) + original-order float4 (x, y, z, spos)
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <vector>

#include "gicp_internal.cuh"

#ifndef GICP_AUTO_OCC
#define GICP_AUTO_OCC 8.0  // target point-weighted voxel occupancy of the automatic cell
#endif

namespace gicp {
namespace {

__device__ __forceinline__ int f2ord(float f) {
    int i = __float_as_int(f);
    return i >= 0 ? i : i ^ 0x7fffffff;
}
inline float ord2f_host(int i) {
    int j = i >= 0 ? i : i ^ 0x7fffffff;
    float f;
    memcpy(&f, &j, 4);
    return f;
}

// out[0..2] = min (ordered ints), out[3..5] = max, out[6] = non-finite count
__global__ void k_bbox(const float* __restrict__ xyz, int64_t n, int* __restrict__ out) {
    int mn[3] = {INT_MAX, INT_MAX, INT_MAX}, mx[3] = {INT_MIN, INT_MIN, INT_MIN};
    int bad = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            float v = xyz[3 * i + a];
            if (!isfinite(v)) {
                bad = 1;
                continue;
            }
            int o = f2ord(v);
            mn[a] = min(mn[a], o);
            mx[a] = max(mx[a], o);
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            mn[a] = min(mn[a], __shfl_xor_sync(0xffffffffu, mn[a], off));
            mx[a] = max(mx[a], __shfl_xor_sync(0xffffffffu, mx[a], off));
        }
        bad |= __shfl_xor_sync(0xffffffffu, bad, off);
    }
    // block reduce, then one set of atomics per block (same-address atomics from
    // every warp would serialise at the L2)
    __shared__ int sh[32][7];
    const int wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if ((threadIdx.x & 31) == 0) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            sh[wid][a] = mn[a];
            sh[wid][3 + a] = mx[a];
        }
        sh[wid][6] = bad;
    }
    __syncthreads();
    if (threadIdx.x < 7) {
        const int c = threadIdx.x;
        int v = sh[0][c];
        for (int w = 1; w < nw; ++w) v = c < 3 ? min(v, sh[w][c]) : (c < 6 ? max(v, sh[w][c]) : (v | sh[w][c]));
        if (c < 3)
            atomicMin(out + c, v);
        else if (c < 6)
            atomicMax(out + c, v);
        else if (v)
            atomicAdd(out + 6, 1);
    }
}

__global__ void k_keys(const float* __restrict__ xyz, int64_t n, Grid g, unsigned long long* __restrict__ keys,
                       int* __restrict__ vals) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float x = xyz[3 * i], y = xyz[3 * i + 1], z = xyz[3 * i + 2];
    int cx = cell_coord(x, g.ox, g.inv_cell), cy = cell_coord(y, g.oy, g.inv_cell), cz = cell_coord(z, g.oz, g.inv_cell);
    cx = min(max(cx, 0), g.nx - 1);  // cannot trigger (monotone cell map); defensive
    cy = min(max(cy, 0), g.ny - 1);
    cz = min(max(cz, 0), g.nz - 1);
    keys[i] = cell_key(cx, cy, cz);
    vals[i] = (int)i;
}

// occupied voxels per level (warp reduce -> block smem counters -> one global
// atomic per level per block)
__global__ void k_level_count(const unsigned long long* __restrict__ keys, int64_t n, int L, int* __restrict__ cnt) {
    __shared__ int sc[kMaxLevels];
    if (threadIdx.x < kMaxLevels) sc[threadIdx.x] = 0;
    __syncthreads();
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const unsigned long long k = i < n ? keys[i] : 0ull;
    const unsigned long long kp = (i > 0 && i < n) ? keys[i - 1] : ~0ull;
    for (int l = 0; l < L; ++l) {
        const int head = (i < n) && (i == 0 || (k >> (3 * l)) != (kp >> (3 * l)));
        const int c = __reduce_add_sync(0xffffffffu, head);
        if ((threadIdx.x & 31) == 0 && c) atomicAdd(&sc[l], c);
    }
    __syncthreads();
    if (threadIdx.x < L && sc[threadIdx.x]) atomicAdd(cnt + threadIdx.x, sc[threadIdx.x]);
}

// sum over level-0 runs of (run length)^2 (the point-weighted mean occupancy
// times n), for the automatic cell size
__global__ void k_runlen2(const unsigned long long* __restrict__ keys, int64_t n,
                          unsigned long long* __restrict__ out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    unsigned long long v = 0;
    if (i < n && (i == 0 || keys[i - 1] != keys[i])) {
        int64_t e = i + 1;
        while (e < n && keys[e] == keys[i]) ++e;
        v = (unsigned long long)(e - i) * (unsigned long long)(e - i);
    }
    v = __reduce_add_sync(0xffffffffu, (unsigned)min(v, 0xffffffffull));
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(out, v);
}

struct LevelSet {
    Grid lv[kMaxLevels];
    int n;
};

// run heads of every level insert their voxel (key >> 3l, start); level-0 heads
// are also appended to a compact list (for the adjacency kernel)
__global__ void k_cells(const unsigned long long* __restrict__ keys, int64_t n, LevelSet ls, int* __restrict__ nheads,
                        int* __restrict__ heads, int* __restrict__ nheads1, int* __restrict__ heads1) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const bool in = i < n;
    const unsigned long long k = in ? keys[i] : 0ull;
    const unsigned long long kp = (in && i > 0) ? keys[i - 1] : ~0ull;
    const bool h0 = in && (i == 0 || kp != k);
    const bool h1 = in && ls.n > 1 && (i == 0 || (kp >> 3) != (k >> 3));
    {
        // compact head lists of levels 0 and 1: warp ballots, one atomic per list
        // per BLOCK (a counter hit by every warp would serialise at the L2)
        __shared__ int wc[2][32];
        __shared__ int bb[2];
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
        const unsigned m0 = __ballot_sync(0xffffffffu, h0), m1 = __ballot_sync(0xffffffffu, h1);
        if (lane == 0) {
            wc[0][wid] = __popc(m0);
            wc[1][wid] = __popc(m1);
        }
        __syncthreads();
        if (threadIdx.x < 2) {
            int t = 0;
            for (int w = 0; w < nw; ++w) {
                const int c = wc[threadIdx.x][w];
                wc[threadIdx.x][w] = t;
                t += c;
            }
            bb[threadIdx.x] = t ? atomicAdd(threadIdx.x == 0 ? nheads : nheads1, t) : 0;
        }
        __syncthreads();
        const unsigned lt = (1u << lane) - 1;
        if (h0) heads[bb[0] + wc[0][wid] + __popc(m0 & lt)] = (int)i;
        if (h1) heads1[bb[1] + wc[1][wid] + __popc(m1 & lt)] = (int)i;
    }
    if (!in) return;
    for (int l = 0; l < ls.n; ++l) {
        const Grid& g = ls.lv[l];
        const int sh = 3 * l;
        const unsigned long long key = k >> sh;
        if (i != 0 && (kp >> sh) == key) break;  // not a head here => not a head at coarser levels
        HashEntry* H = const_cast<HashEntry*>(g.hash);
        unsigned long long h = hash_slot(g, key);
        while (true) {
            unsigned long long prev = atomicCAS(&H[h].key, kEmptyKey, key);
            if (prev == kEmptyKey) {
                H[h].start = (int)i;
                break;
            }
            h = (h + 1) & g.hmask;
        }
    }
}

__global__ void k_set_int(int* p, int v) { *p = v; }

// tile_of[p] = t for every point p of tile t (one warp per tile)
__global__ void k_tile_of(const int* __restrict__ tiles, int64_t nt, int* __restrict__ tile_of) {
    const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    if (w >= nt) return;
    const int a = tiles[w], b = tiles[w + 1];
    for (int p = a + (int)(threadIdx.x & 31); p < b; p += 32) tile_of[p] = (int)w;
}

// run tails of every level write the end of their voxel
__global__ void k_cell_ends(const unsigned long long* __restrict__ keys, int64_t n, LevelSet ls) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const unsigned long long k = keys[i];
    const unsigned long long kn = i + 1 < n ? keys[i + 1] : ~0ull;
    for (int l = 0; l < ls.n; ++l) {
        const Grid& g = ls.lv[l];
        const int sh = 3 * l;
        const unsigned long long key = k >> sh;
        if (i + 1 < n && (kn >> sh) == key) break;
        HashEntry* H = const_cast<HashEntry*>(g.hash);
        unsigned long long h = hash_slot(g, key);
        while (H[h].key != key) h = (h + 1) & g.hmask;
        H[h].end = (int)(i + 1);
    }
}

__global__ void k_scatter(const float* __restrict__ xyz, const int* __restrict__ perm, int64_t n,
                          float4* __restrict__ pts, float4* __restrict__ pts_orig) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int j = perm[i];
    const float x = xyz[3 * (int64_t)j], y = xyz[3 * (int64_t)j + 1], z = xyz[3 * (int64_t)j + 2];
    pts[i] = make_float4(x, y, z, __int_as_float(j));
    pts_orig[j] = make_float4(x, y, z, __int_as_float((int)i));
}

// Level-0 voxel adjacency lists: for every occupied voxel, its
// non-empty voxels among the 27 around it, nearest-first, as (start, end) ranges
// of pts packed with the offset code (adj_pack, gicp_internal.cuh). A query in an
// occupied voxel reads this shared list instead of probing the hash 27 times.
// nearest-first neighbour order (own, 6 faces, 12 edges, 8 corners):
//   (0,0,0) (-1,0,0) (1,0,0) (0,-1,0) (0,1,0) (0,0,-1) (0,0,1) (-1,-1,0) (1,-1,0)
//   (-1,1,0) (1,1,0) (-1,0,-1) (1,0,-1) (-1,0,1) (1,0,1) (0,-1,-1) (0,1,-1) (0,-1,1)
//   (0,1,1) (-1,-1,-1) (1,-1,-1) (-1,1,-1) (1,1,-1) (-1,-1,1) (1,-1,1) (-1,1,1) (1,1,1)

// one warp per occupied level-0 voxel (compact head list): lane c < 27 probes
// neighbour c (27 independent probes in flight per warp); the non-empty ones are
// compacted in nearest-first order with a ballot and appended at an offset the
// BLOCK reserves with one atomic (a single global counter hit once per warp
// serialises at the L2: ~0.5 ns per atomic x 2.6e5 voxels); the list ORDER in
// memory is scheduling-dependent, the list of every voxel is not; (offset,
// count) is stored at the voxel's first point.
constexpr int kAdjBlock = 256;
__global__ void __launch_bounds__(kAdjBlock) k_adjacency(Grid g, int shift, const unsigned long long* __restrict__ keys,
                                                          const int* __restrict__ heads, const int* __restrict__ nheads,
                                                          int* __restrict__ total, int2* __restrict__ oc,
                                                          int2* __restrict__ rng_out, int* __restrict__ overflow) {
    __shared__ int wcnt[kAdjBlock / 32];
    __shared__ int bbase;
    const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const bool valid = w < *nheads;  // warp-uniform; every warp reaches the barriers
    // lane c < 27 takes neighbour c of the nearest-first order above, read
    // from three packed immediates (6-bit codes adj_pack uses) -- a per-lane index
    // into __constant__ memory would serialise 27 ways
    const unsigned long long W = lane < 10 ? 0x612425159456515ull : (lane < 20 ? 0x2984906690611aull : 0x2aa2280a202ull);
    const unsigned code = (unsigned)(W >> (6 * (lane % 10))) & 63u;
    const int dx = (int)(code & 3u) - 1, dy = (int)((code >> 2) & 3u) - 1, dz = (int)((code >> 4) & 3u) - 1;
    int head = 0;
    int2 r = make_int2(0, 0);
    if (valid && lane < 27) {
        head = heads[w];
        // neighbour key by dilated-integer increments of the voxel's Morton key; a
        // step off the grid yields a key no voxel has (empty lookup)
        const unsigned long long key = keys[head] >> shift;
        const unsigned long long MX = 0x1249249249249249ull, MY = MX << 1, MZ = MX << 2;
        auto step = [](unsigned long long k, unsigned long long M, int d) {
            return d < 0 ? ((k - 1ull) & M) : (d > 0 ? (((k | ~M) + 1ull) & M) : k);
        };
        const unsigned long long nk = step(key & MX, MX, dx) | step(key & MY, MY, dy) | step(key & MZ, MZ, dz);
        r = hash_find(g, nk);
    } else if (valid) {
        head = heads[w];
    }
    const bool ne = lane < 27 && r.y > r.x;
    const unsigned mask = __ballot_sync(0xffffffffu, ne);
    const int cnt = __popc(mask);
    if (lane == 0) wcnt[wid] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int i = 0; i < kAdjBlock / 32; ++i) {
            const int c = wcnt[i];
            wcnt[i] = t;
            t += c;
        }
        bbase = t > 0 ? atomicAdd(total, t) : 0;
    }
    __syncthreads();
    const int base = bbase + wcnt[wid];
    if (ne) {
        const int o = base + __popc(mask & ((1u << lane) - 1));
        const int c = r.y - r.x;
        if (c > kAdjMaxCount) atomicOr(overflow, 1);  // count does not fit the packing: no lists
        rng_out[o] = make_int2(r.x, (int)adj_pack(c, dx, dy, dz));
    }
    if (valid && lane == 0) oc[head] = make_int2(base, cnt);
}

__global__ void k_fill_hash(HashEntry* H, int64_t cap) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < cap) {
        H[i].key = kEmptyKey;
        H[i].start = 0;
        H[i].end = 0;
    }
}

struct DevBuf {
    void* p = nullptr;
    cudaStream_t s = nullptr;
    ~DevBuf() {
        if (p) cudaFreeAsync(p, s);
    }
};

int alloc_async(DevBuf& b, size_t bytes, cudaStream_t s) {
    b.s = s;
    cudaError_t e = cudaMallocAsync(&b.p, bytes ? bytes : 16, s);
    if (e != cudaSuccess) {
        cudaGetLastError();
        b.p = nullptr;
        return set_error(GICP_ENOMEM, "device allocation of " + std::to_string(bytes) + " bytes failed");
    }
    return GICP_OK;
}

unsigned grid_for(int64_t n, int block) { return (unsigned)((n + block - 1) / block); }

int bits_for(int dim) {
    int b = 0;
    while ((1 << b) < dim) ++b;
    return b;
}

int make_grid(const float mn[3], const float mx[3], float cell, Grid* g) {
    if (!(cell > 0.0f) || !std::isfinite(cell)) return set_error(GICP_EINVAL, "cell_size must be finite and > 0");
    g->ox = mn[0];
    g->oy = mn[1];
    g->oz = mn[2];
    g->cell = cell;
    volatile float inv = 1.0f / cell;
    g->inv_cell = inv;
    int dims[3];
    for (int a = 0; a < 3; ++a) {
        volatile float d = mx[a] - mn[a];
        volatile float t = d * g->inv_cell;
        double c = std::floor((double)t);
        if (!(c + 1 < kMaxAxisCells))  // < 2^21: a +1 step off the grid never wraps the Morton key
            return set_error(GICP_ERANGE, "voxel grid exceeds 2^21 cells on an axis; increase cell_size");
        dims[a] = (int)c + 1;
    }
    g->nx = dims[0];
    g->ny = dims[1];
    g->nz = dims[2];
    // point-to-voxel assignment error: the map x -> fl(fl(x - o) * inv) carries at
    // most ~3 ulp relative error of |x - o| / cell (cell units), plus fl(1/cell);
    // 8 u (E + cell) + 1e-6 cell bounds it with margin (DESIGN.md §kNN stop rule).
    double E = 0.0;
    for (int a = 0; a < 3; ++a) E = std::fmax(E, (double)mx[a] - (double)mn[a]);
    g->slack = (float)(8.0 * std::ldexp(1.0, -24) * (E + cell) + 1e-6 * cell);
    g->level = 0;
    return GICP_OK;
}

Grid level_grid(const Grid& g0, int l, double E) {
    Grid g = g0;
    g.level = l;
    g.cell = std::ldexp(g0.cell, l);
    g.inv_cell = std::ldexp(g0.inv_cell, -l);  // exact power-of-two scaling
    g.nx = ((g0.nx - 1) >> l) + 1;
    g.ny = ((g0.ny - 1) >> l) + 1;
    g.nz = ((g0.nz - 1) >> l) + 1;
    g.slack = (float)(8.0 * std::ldexp(1.0, -24) * (E + g.cell) + 1e-6 * g.cell);
    return g;
}

// sort (Morton key, i) pairs on the bits in use
int sort_keys(const float* xyz, int64_t n, const Grid& g, cudaStream_t s, DevBuf& keys_out, DevBuf& perm_out) {
    DevBuf keys_in, vals_in, temp;
    int rc;
    if ((rc = alloc_async(keys_in, n * 8, s)) || (rc = alloc_async(vals_in, n * 4, s)) ||
        (rc = alloc_async(keys_out, n * 8, s)) || (rc = alloc_async(perm_out, n * 4, s)))
        return rc;
    k_keys<<<grid_for(n, 256), 256, 0, s>>>(xyz, n, g, (unsigned long long*)keys_in.p, (int*)vals_in.p);
    const int bits = std::max(1, 3 * std::max(bits_for(g.nx), std::max(bits_for(g.ny), bits_for(g.nz))));
    size_t temp_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, (unsigned long long*)keys_in.p,
                                    (unsigned long long*)keys_out.p, (int*)vals_in.p, (int*)perm_out.p, (int)n, 0,
                                    bits, s);
    if ((rc = alloc_async(temp, temp_bytes, s))) return rc;
    return check_cuda(cub::DeviceRadixSort::SortPairs(temp.p, temp_bytes, (unsigned long long*)keys_in.p,
                                                      (unsigned long long*)keys_out.p, (int*)vals_in.p,
                                                      (int*)perm_out.p, (int)n, 0, bits, s),
                      "radix sort");
}

}  // namespace

int build_index(const float* xyz, int64_t n, float cell_size, cudaStream_t s, gicp_index* out) {
    int rc;
    DevBuf bb;
    if ((rc = alloc_async(bb, 16 * sizeof(int), s))) return rc;
    int init[8] = {INT_MAX, INT_MAX, INT_MAX, INT_MIN, INT_MIN, INT_MIN, 0, 0};
    if ((rc = write_small(bb.p, init, sizeof(init), s))) return rc;
    k_bbox<<<(unsigned)std::min<int64_t>(grid_for(n, 256), 148 * 8), 256, 0, s>>>(xyz, n, (int*)bb.p);
    int res[8];
    if ((rc = read_small(res, bb.p, sizeof(res), s))) return rc;
    if (res[6] != 0) return set_error(GICP_EINVAL, "non-finite coordinate in the target cloud");
    float mn[3], mx[3];
    for (int a = 0; a < 3; ++a) {
        mn[a] = ord2f_host(res[a]);
        mx[a] = ord2f_host(res[3 + a]);
    }
    double E = 0.0;
    for (int a = 0; a < 3; ++a) E = std::fmax(E, (double)mx[a] - (double)mn[a]);
    Grid g{};
    if (cell_size == 0.0f) {
        // automatic: trial grid at E/1024; pick the cell so that the point-weighted
        // median voxel occupancy is ~8 (occupancy ~ cell^2 on sampled surfaces).
        // Sparser regions are served by the coarser pyramid levels.
        const float trial = E > 0 ? (float)(E / 1024.0) : 1.0f;
        if ((rc = make_grid(mn, mx, trial, &g))) return rc;
        DevBuf k1, p1, acc;
        if ((rc = sort_keys(xyz, n, g, s, k1, p1))) return rc;
        if ((rc = alloc_async(acc, 16, s))) return rc;
        if ((rc = check_cuda(cudaMemsetAsync(acc.p, 0, 16, s), "memset"))) return rc;
        k_runlen2<<<grid_for(n, 256), 256, 0, s>>>((unsigned long long*)k1.p, n, (unsigned long long*)acc.p);
        unsigned long long sum2 = 0;
        if ((rc = read_small(&sum2, acc.p, 8, s))) return rc;
        // point-weighted mean voxel occupancy at the trial cell; aim at ~12
        const double med = std::max(1.0, (double)sum2 / (double)n) / 1.5;
        cell_size = (float)(trial * std::sqrt(GICP_AUTO_OCC / med));
        if (!(cell_size > 0.0f) || !std::isfinite(cell_size)) cell_size = 1.0f;
    }
    if ((rc = make_grid(mn, mx, cell_size, &g))) return rc;

    DevBuf keys, perm, cnt;
    if ((rc = sort_keys(xyz, n, g, s, keys, perm))) return rc;
    // pyramid depth: until the 27-voxel cube covers the grid, at most kMaxLevels
    int L = 1;
    while (L < kMaxLevels) {
        const Grid gl = level_grid(g, L - 1, E);
        if (gl.nx <= 3 && gl.ny <= 3 && gl.nz <= 3) break;
        ++L;
    }
    if ((rc = alloc_async(cnt, kMaxLevels * sizeof(int), s))) return rc;
    if ((rc = check_cuda(cudaMemsetAsync(cnt.p, 0, kMaxLevels * sizeof(int), s), "memset"))) return rc;
    k_level_count<<<grid_for(n, 256), 256, 0, s>>>((unsigned long long*)keys.p, n, L, (int*)cnt.p);
    int counts[kMaxLevels] = {0};
    if ((rc = read_small(counts, cnt.p, sizeof(counts), s))) return rc;

    gicp_index_s* idx = new gicp_index_s();
    idx->n = n;
    idx->n_levels = L;
    idx->n_cells = counts[0];
    idx->stream = s;
    cudaGetDevice(&idx->device);
    int64_t total_cap = 0;
    for (int l = 0; l < L; ++l) {
        int hb = 1;
        while ((1ll << hb) < 2 * (int64_t)std::max(counts[l], 1)) ++hb;
        idx->lv[l] = level_grid(g, l, E);
        idx->lv[l].hbits = hb;
        idx->lv[l].hmask = (1ull << hb) - 1;
        idx->hash_cap[l] = 1ll << hb;
        total_cap += 1ll << hb;
    }
    auto fail = [&](int code) {
        if (idx->pts) cudaFreeAsync(idx->pts, s);
        if (idx->pts_orig) cudaFreeAsync(idx->pts_orig, s);
        if (idx->hash_mem) cudaFreeAsync(idx->hash_mem, s);
        if (idx->adj_oc) cudaFreeAsync(idx->adj_oc, s);
        if (idx->adj_rng) cudaFreeAsync(idx->adj_rng, s);
        if (idx->adj_oc1) cudaFreeAsync(idx->adj_oc1, s);
        if (idx->adj_rng1) cudaFreeAsync(idx->adj_rng1, s);
        if (idx->tiles1) cudaFreeAsync(idx->tiles1, s);
        if (idx->tile_of) cudaFreeAsync(idx->tile_of, s);
        delete idx;
        return code;
    };
    if (cudaMallocAsync(&idx->pts, n * sizeof(float4), s) != cudaSuccess ||
        cudaMallocAsync(&idx->pts_orig, n * sizeof(float4), s) != cudaSuccess ||
        cudaMallocAsync(&idx->hash_mem, total_cap * sizeof(HashEntry), s) != cudaSuccess) {
        cudaGetLastError();
        return fail(set_error(GICP_ENOMEM, "index allocation failed"));
    }
    idx->device_bytes = n * 2 * (int64_t)sizeof(float4) + total_cap * (int64_t)sizeof(HashEntry);
    k_fill_hash<<<grid_for(total_cap, 256), 256, 0, s>>>(idx->hash_mem, total_cap);
    int64_t off = 0;
    LevelSet ls;
    ls.n = L;
    for (int l = 0; l < L; ++l) {
        idx->lv[l].hash = idx->hash_mem + off;
        off += idx->hash_cap[l];
        ls.lv[l] = idx->lv[l];
    }
    DevBuf headbuf;
    const int64_t n1 = L > 1 ? counts[1] : 0;
    if ((rc = alloc_async(headbuf, (counts[0] + n1 + 8) * sizeof(int), s))) return fail(rc);
    int* nheads = (int*)headbuf.p;  // [0] level-0 heads, [1] level-1 heads
    int* heads = nheads + 8;
    int* heads1 = heads + counts[0];
    if ((rc = check_cuda(cudaMemsetAsync(nheads, 0, 2 * sizeof(int), s), "memset"))) return fail(rc);
    k_cells<<<grid_for(n, 256), 256, 0, s>>>((unsigned long long*)keys.p, n, ls, nheads, heads, nheads + 1, heads1);
    k_cell_ends<<<grid_for(n, 256), 256, 0, s>>>((unsigned long long*)keys.p, n, ls);
    if (L > 1) {
        // the level-1 voxels in sorted (Morton) order: their first points, then n
        if (cudaMallocAsync(&idx->tiles1, (n1 + 1) * sizeof(int), s) != cudaSuccess) {
            cudaGetLastError();
            return fail(set_error(GICP_ENOMEM, "tile list allocation failed"));
        }
        idx->n_tiles1 = n1;
        idx->device_bytes += (n1 + 1) * (int64_t)sizeof(int);
        const int bits = std::max(1, bits_for((int)std::min<int64_t>(n, INT_MAX)));
        size_t tb = 0;
        cub::DeviceRadixSort::SortKeys(nullptr, tb, heads1, idx->tiles1, (int)n1, 0, bits, s);
        DevBuf tmp;
        if ((rc = alloc_async(tmp, tb, s))) return fail(rc);
        cub::DeviceRadixSort::SortKeys(tmp.p, tb, heads1, idx->tiles1, (int)n1, 0, bits, s);
        k_set_int<<<1, 1, 0, s>>>(idx->tiles1 + n1, (int)n);
        if (cudaMallocAsync(&idx->tile_of, n * sizeof(int), s) != cudaSuccess) {
            cudaGetLastError();
            return fail(set_error(GICP_ENOMEM, "tile map allocation failed"));
        }
        idx->device_bytes += n * (int64_t)sizeof(int);
        k_tile_of<<<grid_for(n1 * 32, 256), 256, 0, s>>>(idx->tiles1, n1, idx->tile_of);
    }
    k_scatter<<<grid_for(n, 256), 256, 0, s>>>(xyz, (int*)perm.p, n, idx->pts, idx->pts_orig);
    if ((rc = check_cuda(cudaGetLastError(), "build kernels"))) return fail(rc);
    int adj_overflow = 0;
    {
        // adjacency lists of levels 0 and 1, one pass each (<= 27 entries per voxel)
        DevBuf tot;
        if ((rc = alloc_async(tot, 32, s))) return fail(rc);
        if ((rc = check_cuda(cudaMemsetAsync(tot.p, 0, 32, s), "memset"))) return fail(rc);
        for (int l = 0; l < std::min(L, 2); ++l) {
            int2*& oc = l == 0 ? idx->adj_oc : idx->adj_oc1;
            int2*& rng = l == 0 ? idx->adj_rng : idx->adj_rng1;
            const int64_t nv = std::max(counts[l], 1);
            if (cudaMallocAsync(&oc, n * sizeof(int2), s) != cudaSuccess ||
                cudaMallocAsync(&rng, 27 * nv * sizeof(int2), s) != cudaSuccess) {
                cudaGetLastError();
                return fail(set_error(GICP_ENOMEM, "adjacency allocation failed"));
            }
            idx->adj_cap[l] = 27 * nv;
            // per level: [2l] output counter, [1] overflow flag (shared)
            k_adjacency<<<grid_for(nv * 32, kAdjBlock), kAdjBlock, 0, s>>>(
                idx->lv[l], 3 * l, (unsigned long long*)keys.p, l == 0 ? heads : heads1, nheads + l,
                (int*)tot.p + 2 * l, oc, rng, (int*)tot.p + 1);
            idx->device_bytes += n * 8 + 27 * nv * 8;
            if ((rc = check_cuda(cudaGetLastError(), "adjacency kernel"))) return fail(rc);
        }
        if ((rc = read_small(&adj_overflow, (int*)tot.p + 1, sizeof(int), s))) return fail(rc);
    }
    if ((rc = check_cuda(cudaStreamSynchronize(s), "build"))) return fail(rc);
    if (adj_overflow) {  // a voxel too full for the packed entry: queries probe the hash instead
        for (int2** p : {&idx->adj_oc, &idx->adj_rng, &idx->adj_oc1, &idx->adj_rng1}) {
            if (*p) cudaFreeAsync(*p, s);
            *p = nullptr;
        }
    }
    *out = idx;
    return GICP_OK;
}

}  // namespace gicp
