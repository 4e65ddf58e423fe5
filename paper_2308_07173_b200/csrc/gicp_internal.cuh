// gicp_internal.cuh -- shared device-side definitions of libgicp_b200 (not installed).
//
// Data layout in HBM:
//   pts       float4[n]  points sorted by the level-0 Morton voxel key:
//                        (x, y, z, bitcast(original index)).
//   pts_orig  float4[n]  points in original order: (x, y, z, bitcast(sorted position)).
//   levels    a voxel pyramid, cell_l = cell_0 * 2^l, common origin. Level-l voxel
//             keys are the level-0 Morton keys >> 3l, so every level-l voxel is a
//             contiguous range of `pts` and one sorted array serves all levels.
//             Per level an open-addressing hash {key, start, end} (16 B, one
//             LDG.128 per probe), capacity pow2 >= 2 x occupied voxels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/gicp.h"

#define GICP_HD __host__ __device__ __forceinline__
#define GICP_API extern "C" __attribute__((visibility("default")))

namespace gicp {

constexpr uint64_t kEmptyKey = ~0ull;
constexpr int kMaxAxisCells = 1 << 21;
constexpr int kMaxLevels = 8;

struct HashEntry {
    unsigned long long key;
    int start;
    int end;
};

// One pyramid level, passed by value to kernels.
struct Grid {
    float ox, oy, oz;   // origin (bounding-box minimum), common to all levels
    float cell;         // voxel edge of this level (m)
    float inv_cell;     // fl32(1 / cell) = fl32(1 / cell_0) * 2^-l exactly
    int nx, ny, nz;     // voxels per axis at this level
    float slack;        // conservative geometric slack (m), DESIGN.md §kNN stop rule
    int level;
    int hbits;          // log2(hash capacity)
    unsigned long long hmask;
    const HashEntry* hash;
};

// Cell coordinate along one axis: floor(fl32(fl32(x - o) * inv)). The SAME
// function assigns index points and queries (DESIGN.md §kNN exactness). Because
// inv_l = inv_0 * 2^-l exactly, cell_l(x) == cell_0(x) >> l.
__device__ __forceinline__ int cell_coord(float x, float o, float inv) {
    float t = __fmul_rn(__fsub_rn(x, o), inv);
    t = fminf(fmaxf(t, -1.0e9f), 1.0e9f);
    return (int)floorf(t);
}

// 21-bit Morton spreading
GICP_HD unsigned long long spread3(unsigned x) {
    unsigned long long v = x & 0x1fffffu;
    v = (v | v << 32) & 0x1f00000000ffffull;
    v = (v | v << 16) & 0x1f0000ff0000ffull;
    v = (v | v << 8) & 0x100f00f00f00f00full;
    v = (v | v << 4) & 0x10c30c30c30c30c3ull;
    v = (v | v << 2) & 0x1249249249249249ull;
    return v;
}

GICP_HD unsigned long long cell_key(int cx, int cy, int cz) {
    return spread3((unsigned)cx) | (spread3((unsigned)cy) << 1) | (spread3((unsigned)cz) << 2);
}

GICP_HD unsigned long long hash_slot(const Grid& g, unsigned long long key) {
    return (key * 0x9E3779B97F4A7C15ull) >> (64 - g.hbits);
}

// [start, end) of the voxel with Morton key `key` at level g, or an empty range.
// Linear probing, two slots per step: both loads are issued together, so a probe
// chain costs half as many dependent round trips to L2.
__device__ __forceinline__ int2 hash_find(const Grid& g, unsigned long long key) {
    const int4* __restrict__ H = reinterpret_cast<const int4*>(g.hash);
    unsigned long long h = hash_slot(g, key);
    while (true) {
        const int4 a = __ldg(H + h), b = __ldg(H + ((h + 1) & g.hmask));
        const unsigned long long ka = (unsigned long long)(unsigned)a.x | ((unsigned long long)(unsigned)a.y << 32);
        const unsigned long long kb = (unsigned long long)(unsigned)b.x | ((unsigned long long)(unsigned)b.y << 32);
        if (ka == key) return make_int2(a.z, a.w);
        if (ka == kEmptyKey) return make_int2(0, 0);
        if (kb == key) return make_int2(b.z, b.w);
        if (kb == kEmptyKey) return make_int2(0, 0);
        h = (h + 2) & g.hmask;
    }
}

// Returns [start, end) of the voxel (cx, cy, cz) of level g in pts, or an empty range.
__device__ __forceinline__ int2 cell_lookup(const Grid& g, int cx, int cy, int cz) {
    if ((unsigned)cx >= (unsigned)g.nx || (unsigned)cy >= (unsigned)g.ny || (unsigned)cz >= (unsigned)g.nz)
        return make_int2(0, 0);
    return hash_find(g, cell_key(cx, cy, cz));
}

// The fp32 squared distance in the fixed order (reading R9):
// dx = qx - px; dy = qy - py; dz = qz - pz; d2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx)).
__device__ __forceinline__ float dist2(float qx, float qy, float qz, float px, float py, float pz) {
    const float dx = __fsub_rn(qx, px);
    const float dy = __fsub_rn(qy, py);
    const float dz = __fsub_rn(qz, pz);
    return __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
}

// per-query geometry relative to its voxel at one level
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

// distance from q to the boundary of the cube of Chebyshev radius R around its
// voxel, minus slack: every unsearched point is farther than this
__device__ __forceinline__ float cube_margin(const QGeom& G, float s, float slack, int R) {
    const float mx = fminf(G.fx + R * s, (R + 1) * s - G.fx);
    const float my = fminf(G.fy + R * s, (R + 1) * s - G.fy);
    const float mz = fminf(G.fz + R * s, (R + 1) * s - G.fz);
    return fminf(mx, fminf(my, mz)) - slack;
}

constexpr float kRel = 1.0f - 1.0f / (1 << 20);  // relative safety on squared bounds

}  // namespace gicp

struct gicp_index_s {
    int64_t n = 0;
    int64_t n_cells = 0;  // occupied level-0 voxels
    int n_levels = 0;
    gicp::Grid lv[gicp::kMaxLevels]{};
    int64_t hash_cap[gicp::kMaxLevels]{};
    float4* pts = nullptr;
    float4* pts_orig = nullptr;
    gicp::HashEntry* hash_mem = nullptr;  // all levels' tables, one allocation
    int2* adj_oc = nullptr;               // [n] (offset, count) of the level-0 adjacency list, at voxel heads
    int2* adj_rng = nullptr;              // neighbour voxels, nearest-first per voxel: {start, count<<6 | code}
    int2* adj_oc1 = nullptr;              // the same lists for level 1 (escalated queries)
    int2* adj_rng1 = nullptr;
    int* tiles1 = nullptr;                // level-1 voxels in sorted order: first point of each, then n
    int64_t n_tiles1 = 0;                 //   (the staging units of the tiled kNN, knn_tile.cuh)
    int* tile_of = nullptr;               // [n] the level-1 voxel (index into tiles1) of each sorted point
    float4* cov_sorted = nullptr;         // attached covariances in sorted order (2 x float4 per point)
    float4* vox_mu = nullptr;             // VGICP: per level-0 voxel, at its head: mean - first point (xyz), N (w)
    float4* vox_cov = nullptr;            // VGICP: mean covariance of the voxel's points (2 x float4 at the head)
    const float* vox_attached = nullptr;  // the covariance array the voxel statistics came from
    const float* cov_attached = nullptr;  // the caller's original-order array they were copied from
    int device = 0;
    cudaStream_t stream = nullptr;  // build stream: device memory is pool-allocated on it
    int64_t device_bytes = 0;
    int64_t adj_cap[2] = {0, 0};  // int2 entries of adj_rng / adj_rng1
};

namespace gicp {

// thread-local last-error plumbing (api.cu)
int set_error(int code, const std::string& msg);
int check_cuda(cudaError_t e, const char* what);

// launchers implemented in the .cu files
int build_index(const float* xyz, int64_t n, float cell_size, cudaStream_t s, gicp_index* out);
int launch_knn_self(const gicp_index_s* idx, int k, float eps, int32_t* nbr, float* d2, float* cov, cudaStream_t s);
int launch_knn(const gicp_index_s* idx, const float* q, int64_t m, int k, int32_t* nbr, float* d2, cudaStream_t s);
int launch_knn_subset(const gicp_index_s* idx, const float* q, const int* ids, int64_t n_ids, int k, int32_t* nbr,
                      float* d2, cudaStream_t s);
int launch_query_order(const gicp_index_s* idx, const float* q, int64_t m, int* perm, cudaStream_t s);
// kernel-descriptor weighted covariance parameters (gicp_cov_params, device copy)
struct CovKD {
    int kind;
    float sigma, alpha, c;
    int degree;
    float ox, oy, oz;
    int reg;
    float eps;
};
int launch_covariances_kd(const float* xyz, int64_t n, const float* q, const int32_t* nbr, int64_t m, int k,
                          const CovKD& p, float* cov, cudaStream_t s);
int launch_covariances(const float* xyz, int64_t n, const int32_t* nbr, int64_t m, int k, float eps, float* cov,
                       cudaStream_t s);
// preallocated linearize scratch (gicp_align): block partials + done counter
// Packed level-0 adjacency entry (index.cu k_adjacency): x = first point of the
// neighbour voxel in pts, y = (count << 6) | code, code = (dx+1) | (dy+1) << 2 |
// (dz+1) << 4 for the neighbour's offset (dx, dy, dz) in {-1,0,1}^3.
constexpr int kAdjCountShift = 6;
constexpr int kAdjMaxCount = (1 << (31 - kAdjCountShift)) - 1;
__host__ __device__ __forceinline__ unsigned adj_pack(int count, int dx, int dy, int dz) {
    return ((unsigned)count << kAdjCountShift) | (unsigned)(dx + 1) | ((unsigned)(dy + 1) << 2) |
           ((unsigned)(dz + 1) << 4);
}
// squared lower bound of the distance from the query to the neighbour voxel: per
// axis the gap to the face on the offset's side (lo for -1, hi for +1, 0 for 0)
__device__ __forceinline__ float adj_lb2(unsigned w, float lox, float hix, float loy, float hiy, float loz, float hiz) {
    const unsigned bx = w & 3u, by = (w >> 2) & 3u, bz = (w >> 4) & 3u;
    const float gx = bx == 0u ? lox : (bx == 2u ? hix : 0.0f);
    const float gy = by == 0u ? loy : (by == 2u ? hiy : 0.0f);
    const float gz = bz == 0u ? loz : (bz == 2u ? hiz : 0.0f);
    return __fmaf_rn(gz, gz, __fmaf_rn(gy, gy, gx * gx));
}
__device__ __forceinline__ int2 adj_range(int2 e) { return make_int2(e.x, e.x + (int)((unsigned)e.y >> kAdjCountShift)); }

struct Pose {
    double R[9];
    double t[3];
    double c[3];  // pivot of the rotational perturbation (reading R13)
    float Rf[9];
    int active;   // batched: the registration takes part in this launch
    int cur;      // batched: which correspondence buffer is current (0: corr, 1: corr_old)
    int coarse;   // the search's lockstep cube stage on level 1 (kLinCoarse; far-off poses)
};

// batched launches (gicp_linearize_batched / gicp_align_batched): per block
// {registration, block within it, its block count}, point offsets [B+1], poses [B]
struct BatchView {
    const int4* btab = nullptr;
    const int64_t* offs = nullptr;
    const Pose* poses = nullptr;
    const int* ereg = nullptr;  // entry -> its pose (registration); nullptr: one pose per entry
    int n_scans = 1;
    int n_active = 1;
    int out_stride = 0;
    // deferred reduction (gicp_align_batched): the launch's active entries as
    // {first block in the full table, -}; the kernels only write their block partials
    // and k_lin_reduce sums each entry's partials (the same fixed order) afterwards
    const int2* elist = nullptr;
    int n_e = 0;
    const int4* btab_full = nullptr;
};

struct LinScratch {
    unsigned* done;
    double* partials;
    // optional completion signal (gicp_align): after out29 is written, the last
    // block stores `seq` to *flag (host-mapped memory) so the host can spin on it
    volatile unsigned* flag = nullptr;
    unsigned seq = 0;
    // optional correspondence certificates (gicp_align, reading R27): per source
    // point {search point, rho} of the search that produced corr_old (read) and of
    // this launch's corr (written); nullptr: always search
    float4* cache_new = nullptr;
    const float4* cache_old = nullptr;
    // optional split evaluation (GICP_LIN_SPLIT, with certificates): the queue of
    // points that must search ({search point, i | flags}, one per source point) and
    // its device counter
    float4* queue = nullptr;
    float4* queue2 = nullptr;    // the points the first search pass leaves to the full search
    unsigned* qcount = nullptr;  // [4]: queue length, its claim counter, queue2 length, its claim counter
};
constexpr int kLinCorrSpos = 1 << 8;  // internal flag: corr holds sorted positions
constexpr int kLinCoarse = 1 << 10;   // internal flag: single launches set Pose::coarse
constexpr int kLinDual = 1 << 9;      // internal flag: also the trial cost with corr_old (values 29, 30)
constexpr int kLinNV = 31;            // values a DUAL launch reduces per registration
size_t linearize_partials_bytes(int64_t nblocks);
size_t linearize_scratch_bytes(int64_t ns);
int launch_linearize(const float* src, const float* src_cov, int64_t ns, const gicp_index_s* tgt,
                     const float* tgt_cov, const double T[16], const double* pivot, float max_corr_dist, int flags,
                     double* out29, int32_t* corr, cudaStream_t s, const LinScratch* pre = nullptr,
                     const int32_t* corr_old = nullptr);
// the pose block of a launch: R, t (fp64 and fp32 R) and the perturbation pivot
Pose make_pose(const double T[16], const double* pivot);
// lanes per source point in the linearisation (the candidate scan is split
// between them: more warps in flight for the latency-bound 1-NN search)
#ifndef GICP_LIN_TEAM
#define GICP_LIN_TEAM 1  // measured: 2 lanes +15 %, 4 lanes +48 % (the per-warp reductions double)
#endif
// points per linearize block (the fixed partition of every registration)
constexpr int kLinPPB = 256 / GICP_LIN_TEAM;
// one launch over nb blocks: single (bv.btab == nullptr, P) or batched (bv)
int launch_linearize_core(const float* src, const float* src_cov, int64_t ns, const gicp_index_s* tgt,
                          const float* tgt_cov, const Pose& P, float max_corr_dist, int flags, double* out29,
                          int32_t* corr, cudaStream_t s, const LinScratch& scr, const int32_t* corr_old,
                          const BatchView& bv, int64_t nb);
int attach_covariances(gicp_index_s* idx, const float* cov, cudaStream_t s);
int attach_voxels(gicp_index_s* idx, const float* cov, cudaStream_t s);
// Small device<->host transfers of the library's own bookkeeping that bypass the
// copy engines: a caller's bulk cudaMemcpyAsync on another stream would otherwise
// sit in the same DMA queue ahead of them (measured: +0.9 ms on the e2e step with
// a 48 MB download running). read_small: a one-block kernel stores the bytes into
// host-mapped memory, then the stream is synchronised. write_small (<= 256 B):
// the bytes travel as a kernel argument.
int read_small(void* dst, const void* src_dev, size_t bytes, cudaStream_t s);
int write_small(void* dst_dev, const void* src, size_t bytes, cudaStream_t s);
int launch_cluster(const float* xyz, int64_t n, float tol, int min_size, int32_t* label, int64_t* n_clusters,
                   cudaStream_t s);
int launch_ground_filter(const float* xyz, int64_t n, float cell, int min_count, uint8_t* keep, int32_t* count,
                         cudaStream_t s);
size_t vgicp_scratch_bytes(int64_t ns);
int launch_linearize_vgicp(const float* src, const float* src_cov, int64_t ns, const gicp_index_s* tgt,
                           const double T[16], const double* pivot, int mode, int flags, int* base, double* out29,
                           cudaStream_t s, const LinScratch* pre = nullptr);
// sharded linearisation (shard.cu): entry rows -> global chunk table, chunk-ordered combine
int launch_scatter_rows(const double* rows, int E, const int* gid_dev, const int* ereg_dev, const Pose* poses_dev,
                        const int64_t* offs_dev, double* table, cudaStream_t s);
int launch_combine_chunks(const double* table, int B, int nc, int width, double* out, volatile unsigned* flag,
                          unsigned seq, cudaStream_t s);
int launch_compact_btab(const int4* btab, const int2* clist, int nce, int total, int4* ctab, cudaStream_t s);
int sort_source(const float* src, const float* src_cov, int64_t ns, float cell, float* src_p, float* cov_p,
                cudaStream_t s, const int64_t* offs = nullptr, int nseg = 1);

}  // namespace gicp
