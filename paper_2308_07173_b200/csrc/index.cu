// index.cu -- gicp_build_index: uniform voxel grid built by radix sort on cell keys.
//
// Paper: the structure behind "GPU-based nearest points search" (PAPER.md l.413,
// "GPU-hash data structure" l.477); north star: "a uniform voxel grid built by
// radix sort on cell keys". Steps:
//   1. k_bbox      finiteness check + bounding box (block reduce, ordered-int atomics)
//   2. k_keys      key_i = linear voxel id of floor(fl32(fl32(x - o) * inv))
//   3. CUB radix sort (key, i) on only the key bits needed
//   4. k_heads     run boundaries -> voxel start/end, hash insert (atomicCAS)
//   5. k_scatter   sorted float4 (x, y, z, orig) + original-order float4 (x, y, z, spos)
#include <cub/cub.cuh>

#include <cmath>
#include <cstdio>
#include <vector>

#include "gicp_internal.cuh"

namespace gicp {
namespace {

__device__ __forceinline__ int f2ord(float f) {
    int i = __float_as_int(f);
    return i >= 0 ? i : i ^ 0x7fffffff;
}
__host__ __device__ inline float ord2f(int i) {
#ifdef __CUDA_ARCH__
    return __int_as_float(i >= 0 ? i : i ^ 0x7fffffff);
#else
    int j = i >= 0 ? i : i ^ 0x7fffffff;
    float f;
    memcpy(&f, &j, 4);
    return f;
#endif
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
    if ((threadIdx.x & 31) == 0) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            atomicMin(out + a, mn[a]);
            atomicMax(out + 3 + a, mx[a]);
        }
        if (bad) atomicAdd(out + 6, 1);
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
    keys[i] = cell_key(g, cx, cy, cz);
    vals[i] = (int)i;
}

__global__ void k_heads(const unsigned long long* __restrict__ keys, int64_t n, int* __restrict__ head) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    head[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}

// one thread per sorted point; run heads insert their voxel (key, start)
__global__ void k_cells(const unsigned long long* __restrict__ keys, int64_t n, Grid g, HashEntry* __restrict__ H) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const unsigned long long key = keys[i];
    if (i != 0 && keys[i - 1] == key) return;
    unsigned long long h = hash_slot(g, key);
    while (true) {
        unsigned long long prev = atomicCAS(&H[h].key, kEmptyKey, key);
        if (prev == kEmptyKey) {
            H[h].start = (int)i;
            return;
        }
        h = (h + 1) & g.hmask;
    }
}

// run tails write the end of their voxel (O(1) per point for any occupancy)
__global__ void k_cell_ends(const unsigned long long* __restrict__ keys, int64_t n, Grid g, HashEntry* __restrict__ H) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const unsigned long long key = keys[i];
    if (i + 1 < n && keys[i + 1] == key) return;
    unsigned long long h = hash_slot(g, key);
    while (H[h].key != key) h = (h + 1) & g.hmask;
    H[h].end = (int)(i + 1);
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
        return set_error(GICP_ENOMEM, "device allocation of " + std::to_string(bytes) + " bytes failed");
    }
    return GICP_OK;
}

unsigned grid_for(int64_t n, int block) { return (unsigned)((n + block - 1) / block); }

// key bits actually used by the linear voxel id
int key_bits(const Grid& g) {
    unsigned long long total = (unsigned long long)g.nx * g.ny * g.nz;
    int b = 1;
    while (b < 64 && (1ull << b) < total) ++b;
    return b;
}

// sort (key, i) pairs on the key bits in use and count voxels (run heads).
// Leaves sorted keys / permutation in keys_out / perm_out.
int sort_cells(const float* xyz, int64_t n, const Grid& g, cudaStream_t s, DevBuf& keys_out, DevBuf& perm_out,
               int64_t* n_cells_out) {
    DevBuf keys_in, vals_in, temp, cnt, head, t2;
    int rc;
    if ((rc = alloc_async(keys_in, n * 8, s)) || (rc = alloc_async(vals_in, n * 4, s)) ||
        (rc = alloc_async(keys_out, n * 8, s)) || (rc = alloc_async(perm_out, n * 4, s)) ||
        (rc = alloc_async(cnt, 16, s)) || (rc = alloc_async(head, n * 4, s)))
        return rc;
    k_keys<<<grid_for(n, 256), 256, 0, s>>>(xyz, n, g, (unsigned long long*)keys_in.p, (int*)vals_in.p);
    size_t temp_bytes = 0;
    const int bits = key_bits(g);
    cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, (unsigned long long*)keys_in.p,
                                    (unsigned long long*)keys_out.p, (int*)vals_in.p, (int*)perm_out.p, (int)n, 0,
                                    bits, s);
    if ((rc = alloc_async(temp, temp_bytes, s))) return rc;
    if ((rc = check_cuda(cub::DeviceRadixSort::SortPairs(temp.p, temp_bytes, (unsigned long long*)keys_in.p,
                                                         (unsigned long long*)keys_out.p, (int*)vals_in.p,
                                                         (int*)perm_out.p, (int)n, 0, bits, s),
                         "radix sort")))
        return rc;
    k_heads<<<grid_for(n, 256), 256, 0, s>>>((unsigned long long*)keys_out.p, n, (int*)head.p);
    size_t tb = 0;
    cub::DeviceReduce::Sum(nullptr, tb, (int*)head.p, (int*)cnt.p, (int)n, s);
    if ((rc = alloc_async(t2, tb, s))) return rc;
    cub::DeviceReduce::Sum(t2.p, tb, (int*)head.p, (int*)cnt.p, (int)n, s);
    int hc = 0;
    if ((rc = check_cuda(cudaMemcpyAsync(&hc, cnt.p, 4, cudaMemcpyDeviceToHost, s), "D2H"))) return rc;
    if ((rc = check_cuda(cudaStreamSynchronize(s), "build sync"))) return rc;
    *n_cells_out = hc;
    return check_cuda(cudaGetLastError(), "build kernels");
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
        if (c + 1 > kMaxAxisCells)
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
    return GICP_OK;
}

}  // namespace

int build_index(const float* xyz, int64_t n, float cell_size, cudaStream_t s, gicp_index* out) {
    int rc;
    DevBuf bb;
    if ((rc = alloc_async(bb, 8 * sizeof(int), s))) return rc;
    int init[8] = {INT_MAX, INT_MAX, INT_MAX, INT_MIN, INT_MIN, INT_MIN, 0, 0};
    if ((rc = check_cuda(cudaMemcpyAsync(bb.p, init, sizeof(init), cudaMemcpyHostToDevice, s), "H2D"))) return rc;
    {
        unsigned blocks = (unsigned)std::min<int64_t>(grid_for(n, 256), 148 * 8);
        k_bbox<<<blocks, 256, 0, s>>>(xyz, n, (int*)bb.p);
    }
    int res[8];
    if ((rc = check_cuda(cudaMemcpyAsync(res, bb.p, sizeof(res), cudaMemcpyDeviceToHost, s), "D2H"))) return rc;
    if ((rc = check_cuda(cudaStreamSynchronize(s), "bbox"))) return rc;
    if (res[6] != 0) return set_error(GICP_EINVAL, "non-finite coordinate in the target cloud");
    float mn[3], mx[3];
    for (int a = 0; a < 3; ++a) {
        mn[a] = ord2f(res[a]);
        mx[a] = ord2f(res[3 + a]);
    }
    Grid g{};
    if (cell_size == 0.0f) {
        // automatic: trial grid at E/1024, then scale so that occupied voxels hold
        // about 8 points on average (surface sampling: occupancy ~ cell^2).
        float E = std::fmax(mx[0] - mn[0], std::fmax(mx[1] - mn[1], mx[2] - mn[2]));
        float trial = E > 0 ? E / 1024.0f : 1.0f;
        if ((rc = make_grid(mn, mx, trial, &g))) return rc;
        g.hbits = 1;
        DevBuf k1, p1;
        int64_t nc = 0;
        if ((rc = sort_cells(xyz, n, g, s, k1, p1, &nc))) return rc;
        double occ = (double)n / (double)std::max<int64_t>(nc, 1);
        cell_size = (float)(trial * std::sqrt(8.0 / occ));
        if (!(cell_size > 0.0f)) cell_size = 1.0f;
    } else if (!(cell_size > 0.0f) || !std::isfinite(cell_size)) {
        return set_error(GICP_EINVAL, "cell_size must be >= 0 and finite");
    }
    if ((rc = make_grid(mn, mx, cell_size, &g))) return rc;

    g.hbits = 1;
    int64_t ncells = 0;
    DevBuf keys, perm;
    if ((rc = sort_cells(xyz, n, g, s, keys, perm, &ncells))) return rc;
    int hb = 1;
    while ((1ll << hb) < 2 * ncells) ++hb;
    g.hbits = hb;
    g.hmask = (1ull << hb) - 1;
    const int64_t cap = 1ll << hb;

    gicp_index_s* idx = new gicp_index_s();
    idx->n = n;
    idx->g = g;
    idx->hash_cap = cap;
    idx->n_cells = ncells;
    cudaGetDevice(&idx->device);
    auto fail = [&](int code) {
        if (idx->pts) cudaFreeAsync(idx->pts, s);
        if (idx->pts_orig) cudaFreeAsync(idx->pts_orig, s);
        if (idx->hash) cudaFreeAsync(idx->hash, s);
        delete idx;
        return code;
    };
    idx->stream = s;
    if (cudaMallocAsync(&idx->pts, n * sizeof(float4), s) != cudaSuccess ||
        cudaMallocAsync(&idx->pts_orig, n * sizeof(float4), s) != cudaSuccess ||
        cudaMallocAsync(&idx->hash, cap * sizeof(HashEntry), s) != cudaSuccess) {
        cudaGetLastError();
        return fail(set_error(GICP_ENOMEM, "index allocation failed"));
    }
    idx->device_bytes = n * 2 * (int64_t)sizeof(float4) + cap * (int64_t)sizeof(HashEntry);
    {
        k_fill_hash<<<grid_for(cap, 256), 256, 0, s>>>(idx->hash, cap);
        k_cells<<<grid_for(n, 256), 256, 0, s>>>((unsigned long long*)keys.p, n, g, idx->hash);
        k_cell_ends<<<grid_for(n, 256), 256, 0, s>>>((unsigned long long*)keys.p, n, g, idx->hash);
        k_scatter<<<grid_for(n, 256), 256, 0, s>>>(xyz, (int*)perm.p, n, idx->pts, idx->pts_orig);
        if ((rc = check_cuda(cudaStreamSynchronize(s), "build"))) return fail(rc);
    }
    if ((rc = check_cuda(cudaGetLastError(), "build kernels"))) return fail(rc);
    *out = idx;
    return GICP_OK;
}

}  // namespace gicp
