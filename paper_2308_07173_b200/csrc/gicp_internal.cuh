// gicp_internal.cuh -- shared device-side definitions of libgicp_b200 (not installed).
//
// Data layout in HBM:
//   pts       float4[n]  points sorted by voxel key: (x, y, z, bitcast(original index)).
//   pts_orig  float4[n]  points in original order: (x, y, z, bitcast(sorted position)).
//   hash      HashEntry[cap] open addressing, 16 B entries {key, start, end}: one
//             LDG.128 per probe; cap = pow2 >= 2 * occupied voxels (load <= 0.5).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/gicp.h"

#define GICP_HD __host__ __device__ __forceinline__

namespace gicp {

constexpr uint64_t kEmptyKey = ~0ull;
constexpr int kMaxAxisCells = 1 << 21;

struct HashEntry {
    unsigned long long key;
    int start;
    int end;
};

// Grid parameters passed by value to kernels.
struct Grid {
    float ox, oy, oz;   // origin (bounding-box minimum)
    float cell;         // voxel edge (m)
    float inv_cell;     // fl32(1 / cell)
    int nx, ny, nz;     // voxels per axis
    float slack;        // conservative geometric slack (m), see DESIGN.md §kNN stop rule
    int hbits;          // log2(hash capacity)
    unsigned long long hmask;
};

// Cell coordinate along one axis: floor(fl32(fl32(x - o) * inv)). The SAME
// function assigns index points and queries (DESIGN.md §kNN exactness).
__device__ __forceinline__ int cell_coord(float x, float o, float inv) {
    float t = __fmul_rn(__fsub_rn(x, o), inv);
    t = fminf(fmaxf(t, -1.0e9f), 1.0e9f);
    return (int)floorf(t);
}

GICP_HD unsigned long long cell_key(const Grid& g, int cx, int cy, int cz) {
    return ((unsigned long long)cz * (unsigned long long)g.ny + (unsigned long long)cy) * (unsigned long long)g.nx +
           (unsigned long long)cx;
}

GICP_HD unsigned long long hash_slot(const Grid& g, unsigned long long key) {
    return (key * 0x9E3779B97F4A7C15ull) >> (64 - g.hbits);
}

// Returns [start, end) of the voxel (cx, cy, cz) in pts, or an empty range.
__device__ __forceinline__ int2 cell_lookup(const HashEntry* __restrict__ H, const Grid& g, int cx, int cy, int cz) {
    if ((unsigned)cx >= (unsigned)g.nx || (unsigned)cy >= (unsigned)g.ny || (unsigned)cz >= (unsigned)g.nz)
        return make_int2(0, 0);
    const unsigned long long key = cell_key(g, cx, cy, cz);
    unsigned long long h = hash_slot(g, key);
    while (true) {
        const int4 e = __ldg(reinterpret_cast<const int4*>(H) + h);
        const unsigned long long k = (unsigned long long)(unsigned)e.x | ((unsigned long long)(unsigned)e.y << 32);
        if (k == key) return make_int2(e.z, e.w);
        if (k == kEmptyKey) return make_int2(0, 0);
        h = (h + 1) & g.hmask;
    }
}

// The fp32 squared distance in the fixed order (reading R9):
// dx = qx - px; dy = qy - py; dz = qz - pz; d2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx)).
__device__ __forceinline__ float dist2(float qx, float qy, float qz, float px, float py, float pz) {
    const float dx = __fsub_rn(qx, px);
    const float dy = __fsub_rn(qy, py);
    const float dz = __fsub_rn(qz, pz);
    return __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
}

}  // namespace gicp

struct gicp_index_s {
    int64_t n = 0;
    int64_t n_cells = 0;
    gicp::Grid g{};
    float4* pts = nullptr;
    float4* pts_orig = nullptr;
    gicp::HashEntry* hash = nullptr;
    int64_t hash_cap = 0;
    int device = 0;
    cudaStream_t stream = nullptr;  // build stream: device memory is pool-allocated on it
    int64_t device_bytes = 0;
};

namespace gicp {

// thread-local last-error plumbing (api.cu)
int set_error(int code, const std::string& msg);
int check_cuda(cudaError_t e, const char* what);

// launchers implemented in the .cu files
int build_index(const float* xyz, int64_t n, float cell_size, cudaStream_t s, gicp_index* out);
int launch_knn_self(const gicp_index_s* idx, int k, float eps, int32_t* nbr, float* d2, float* cov, cudaStream_t s);
int launch_knn(const gicp_index_s* idx, const float* q, int64_t m, int k, int32_t* nbr, float* d2, cudaStream_t s);
int launch_covariances(const float* xyz, int64_t n, const int32_t* nbr, int64_t m, int k, float eps, float* cov,
                       cudaStream_t s);
int launch_linearize(const float* src, const float* src_cov, int64_t ns, const gicp_index_s* tgt,
                     const float* tgt_cov, const double T[16], float max_corr_dist, int flags, double* out29,
                     int32_t* corr, cudaStream_t s);

}  // namespace gicp
