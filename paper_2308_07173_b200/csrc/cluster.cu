// cluster.cu -- Euclidean cluster extraction ("CUDA-based
// Euclidean distance clustering ... to find cluster C_j", Rusu 2010; SURVEY.md
// §8(f) #4; reading R25).
//
// i ~ j iff d2(p_i, p_j) <= fl32(tol * tol) (the R9 fp32 d2); clusters are the
// connected components, numbered by descending size then smallest member index,
// those below min_size labelled -1.
//   1. a voxel index at cell = tol (1 + 2^-10): every neighbour within tol lies in
//      the 27-voxel cube of the point (level-0 adjacency lists)
//   2. lock-free union-find over sorted positions: for every pair within tol with
//      j > i, link the larger root to the smaller (atomicCAS, retried) -- the final
//      root of a component is its smallest sorted position
//   3. flatten; per root: size, smallest ORIGINAL index (atomicMin)
//   4. one CUB sort of the roots by (n - size, smallest original index) -> rank
//   5. label[original index] = rank of its root, or -1 below min_size
#include <cub/cub.cuh>

#include "gicp_internal.cuh"

namespace gicp {
namespace {

__device__ __forceinline__ int uf_find(const int* __restrict__ par, int x) {
    int p = __ldcg(par + x);
    while (p != x) {
        x = p;
        p = __ldcg(par + x);
    }
    return x;
}

__global__ void k_uf_init(int* par, int64_t n) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) par[i] = (int)i;
}

__global__ void k_uf_link(const float4* __restrict__ pts, int64_t n, Grid g, const int2* __restrict__ adj_oc,
                          const int2* __restrict__ adj_rng, float t2, int* par) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float4 q = pts[i];
    const int cx = cell_coord(q.x, g.ox, g.inv_cell), cy = cell_coord(q.y, g.oy, g.inv_cell),
              cz = cell_coord(q.z, g.oz, g.inv_cell);
    auto visit = [&](int2 r) {
        for (int j = max(r.x, (int)i + 1); j < r.y; ++j) {
            const float4 p = __ldg(pts + j);
            if (!(dist2(q.x, q.y, q.z, p.x, p.y, p.z) <= t2)) continue;
            int a = (int)i, b = j;
            while (true) {
                a = uf_find(par, a);
                b = uf_find(par, b);
                if (a == b) break;
                if (a > b) {
                    const int t = a;
                    a = b;
                    b = t;
                }
                if (atomicCAS(par + b, b, a) == b) break;  // b was still a root: linked
            }
        }
    };
    const int2 own = cell_lookup(g, cx, cy, cz);
    if (adj_oc && own.y > own.x) {
        const int2 oc = __ldg(adj_oc + own.x);
        for (int e = oc.x; e < oc.x + oc.y; ++e) visit(adj_range(__ldg(adj_rng + e)));
    } else {
        for (int dz = -1; dz <= 1; ++dz)
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) visit(cell_lookup(g, cx + dx, cy + dy, cz + dz));
    }
}

__global__ void k_uf_flatten(const float4* __restrict__ pts, int64_t n, int* par, int* __restrict__ size,
                             int* __restrict__ minorig) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int r = uf_find(par, (int)i);
    par[i] = r;
    atomicAdd(size + r, 1);
    atomicMin(minorig + r, __float_as_int(pts[i].w));
}

__global__ void k_root_keys(const int* __restrict__ par, int64_t n, const int* __restrict__ size,
                            const int* __restrict__ minorig, int min_size, unsigned long long* __restrict__ keys,
                            int* __restrict__ vals, int* __restrict__ ncl) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const bool root = par[i] == (int)i && size[i] >= min_size;
    keys[i] = root ? (((unsigned long long)(n - size[i]) << 32) | (unsigned)minorig[i]) : ~0ull;
    vals[i] = (int)i;
    if (root) atomicAdd(ncl, 1);
}

__global__ void k_rank(const unsigned long long* __restrict__ keys, const int* __restrict__ vals, int64_t n,
                       int* __restrict__ rank) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r < n && keys[r] != ~0ull) rank[vals[r]] = (int)r;
}

__global__ void k_label(const float4* __restrict__ pts, int64_t n, const int* __restrict__ par,
                        const int* __restrict__ size, const int* __restrict__ rank, int min_size,
                        int32_t* __restrict__ label) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int r = par[i];
    label[__float_as_int(pts[i].w)] = size[r] >= min_size ? rank[r] : -1;
}

}  // namespace

int launch_cluster(const float* xyz, int64_t n, float tol, int min_size, int32_t* label, int64_t* n_clusters,
                   cudaStream_t s) {
    *n_clusters = 0;
    if (n == 0) return GICP_OK;
    gicp_index idx = nullptr;
    // every neighbour within tol must lie in the point's 27-voxel cube: the voxel edge
    // must exceed tol by the voxel-assignment rounding, which grows with the cloud's
    // extent (the grid's slack, 8u(E + cell)); rebuild once if the first margin is short
    float cell = tol * (1.0f + 1.0f / 1024.0f);
    int rc = build_index(xyz, n, cell, s, &idx);
    if (rc) return rc;
    if (idx->lv[0].slack >= cell - tol) {
        const float c2 = tol + 2.0f * idx->lv[0].slack + tol / 1024.0f;
        gicp_index_free(idx);
        idx = nullptr;
        if ((rc = build_index(xyz, n, c2, s, &idx))) return rc;
        if (idx->lv[0].slack >= idx->lv[0].cell - tol) {
            gicp_index_free(idx);
            return set_error(GICP_ERANGE, "gicp_cluster: tolerance below the grid's rounding slack");
        }
    }
    const volatile float t2v = tol * tol;
    const float t2 = t2v;
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, (unsigned long long*)nullptr, (unsigned long long*)nullptr,
                                    (int*)nullptr, (int*)nullptr, (int)n, 0, 64, s);
    // par | size | minorig | rank | vals_in | vals_out | ncl | keys_in | keys_out | temp
    const size_t ints = 6 * (size_t)n + 4;
    char* buf = nullptr;
    const size_t bytes = ints * 4 + 16 + 2 * (size_t)n * 8 + tb + 64;
    if (cudaMallocAsync((void**)&buf, bytes, s) != cudaSuccess) {
        cudaGetLastError();
        gicp_index_free(idx);
        return set_error(GICP_ENOMEM, "cluster: scratch allocation failed");
    }
    int* par = (int*)buf;
    int* size = par + n;
    int* minorig = size + n;
    int* rank = minorig + n;
    int* vin = rank + n;
    int* vout = vin + n;
    int* ncl = vout + n;
    unsigned long long* kin = (unsigned long long*)(((uintptr_t)(ncl + 4) + 15) & ~(uintptr_t)15);
    unsigned long long* kout = kin + n;
    void* temp = (void*)(((uintptr_t)(kout + n) + 15) & ~(uintptr_t)15);
    const unsigned G = (unsigned)((n + 255) / 256);
    cudaMemsetAsync(size, 0, n * sizeof(int), s);
    cudaMemsetAsync(minorig, 0x7f, n * sizeof(int), s);
    cudaMemsetAsync(ncl, 0, sizeof(int), s);
    k_uf_init<<<G, 256, 0, s>>>(par, n);
    k_uf_link<<<G, 256, 0, s>>>(idx->pts, n, idx->lv[0], idx->adj_oc, idx->adj_rng, t2, par);
    k_uf_flatten<<<G, 256, 0, s>>>(idx->pts, n, par, size, minorig);
    k_root_keys<<<G, 256, 0, s>>>(par, n, size, minorig, min_size, kin, vin, ncl);
    cub::DeviceRadixSort::SortPairs(temp, tb, kin, kout, vin, vout, (int)n, 0, 64, s);
    k_rank<<<G, 256, 0, s>>>(kout, vout, n, rank);
    k_label<<<G, 256, 0, s>>>(idx->pts, n, par, size, rank, min_size, label);
    int h = 0;
    rc = check_cuda(cudaGetLastError(), "cluster kernels");
    if (!rc) rc = read_small(&h, ncl, sizeof(int), s);
    cudaFreeAsync(buf, s);
    gicp_index_free(idx);
    *n_clusters = h;
    return rc;
}

}  // namespace gicp
