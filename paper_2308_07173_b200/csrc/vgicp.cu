// vgicp.cu -- voxelized GICP ("extends and optimizes the
// Voxelized-GICP"; readings R22-R23).
//
// The target's level-0 voxels (the index built with cell = the VGICP
// resolution) carry a Gaussian each: N, mean, and the mean of the points'
// covariances. A source point's correspondences are the voxels of fl32(T p) and
// its 6 face (mode 7) or 26 (mode 27) neighbours -- hash lookups instead of a
// nearest-neighbour search -- and each pair adds N (J^T M J, J^T M d, d^T M d),
// d = mean - T p, M = (Sigma_v + R C_p R^T)^-1.
//
//   k_voxel_stats       one thread per level-0 hash slot: fp64 sums over the
//                       voxel's points -> mean offset (from its first sorted point,
//                       fp32) and mean covariance (fp32), stored at the voxel head
//   k_linearize_vgicp   one thread per source point, PPB = 256 fixed partition,
//                       warp / block / last-block fixed-order fp64 reduction
#include "gicp_internal.cuh"
#include "lin_device.cuh"

namespace gicp {
namespace {

__global__ void k_voxel_stats(const HashEntry* __restrict__ H, int64_t cap, const float4* __restrict__ pts,
                              const float* __restrict__ cov, float4* __restrict__ mu, float4* __restrict__ vcov) {
    const int64_t h = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (h >= cap) return;
    const HashEntry e = H[h];
    if (e.key == kEmptyKey || e.end <= e.start) return;
    const float4 p0 = pts[e.start];
    double s[3] = {0, 0, 0}, c[6] = {0, 0, 0, 0, 0, 0};
    for (int j = e.start; j < e.end; ++j) {
        const float4 p = pts[j];
        s[0] += (double)p.x - (double)p0.x;
        s[1] += (double)p.y - (double)p0.y;
        s[2] += (double)p.z - (double)p0.z;
        const float* cj = cov + 6 * (int64_t)__float_as_int(p.w);
#pragma unroll
        for (int a = 0; a < 6; ++a) c[a] += (double)cj[a];
    }
    const double inv = 1.0 / (double)(e.end - e.start);
    mu[e.start] = make_float4((float)(s[0] * inv), (float)(s[1] * inv), (float)(s[2] * inv), (float)(e.end - e.start));
    vcov[2 * (int64_t)e.start] = make_float4((float)(c[0] * inv), (float)(c[1] * inv), (float)(c[2] * inv),
                                             (float)(c[3] * inv));
    vcov[2 * (int64_t)e.start + 1] = make_float4((float)(c[4] * inv), (float)(c[5] * inv), 0.f, 0.f);
}

constexpr int kVB = 256;  // points per block (the fixed partition)
constexpr int kVNV = 29;

__device__ __forceinline__ double vwarp_sum(double v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
    return v;
}

template <bool ERROR_ONLY, bool REUSE>
__global__ void __launch_bounds__(kVB, 4) k_linearize_vgicp(const float* __restrict__ src,
                                                             const float* __restrict__ src_cov, int64_t ns,
                                                             const float4* __restrict__ pts, Grid g,
                                                             const float4* __restrict__ vmu,
                                                             const float4* __restrict__ vcov, Pose P, int mode,
                                                             int* __restrict__ base,
                                                             double* __restrict__ partials, unsigned* __restrict__ done,
                                                             double* __restrict__ out29) {
    double acc[28];
#pragma unroll
    for (int c = 0; c < 28; ++c) acc[c] = 0.0;
    double cnt = 0.0;
    const int64_t i = (int64_t)blockIdx.x * kVB + threadIdx.x;
    if (i < ns) {
        double pp[3];
        const double px = src[3 * i], py = src[3 * i + 1], pz = src[3 * i + 2];
#pragma unroll
        for (int a = 0; a < 3; ++a)
            pp[a] = __fma_rn(P.R[3 * a + 2], pz, __fma_rn(P.R[3 * a + 1], py, __fma_rn(P.R[3 * a], px, P.t[a])));
        int cx, cy, cz;
        if (REUSE) {  // the pairs of the previous linearisation (reading R23)
            cx = base[3 * i];
            cy = base[3 * i + 1];
            cz = base[3 * i + 2];
        } else {
            cx = cell_coord((float)pp[0], g.ox, g.inv_cell);
            cy = cell_coord((float)pp[1], g.oy, g.inv_cell);
            cz = cell_coord((float)pp[2], g.oz, g.inv_cell);
            if (base) {
                base[3 * i] = cx;
                base[3 * i + 1] = cy;
                base[3 * i + 2] = cz;
            }
        }
        float cp[6];
        {
            const float2* q = reinterpret_cast<const float2*>(src_cov + 6 * i);
            const float2 a = __ldg(q), b = __ldg(q + 1), d = __ldg(q + 2);
            cp[0] = a.x; cp[1] = a.y; cp[2] = b.x; cp[3] = b.y; cp[4] = d.x; cp[5] = d.y;
        }
        // nearest-first offsets: own, 6 faces, 12 edges, 8 corners (reading R22)
        constexpr signed char off[27][3] = {
            {0, 0, 0},   {-1, 0, 0},  {1, 0, 0},   {0, -1, 0},  {0, 1, 0},   {0, 0, -1},  {0, 0, 1},
            {-1, -1, 0}, {1, -1, 0},  {-1, 1, 0},  {1, 1, 0},   {-1, 0, -1}, {1, 0, -1},  {-1, 0, 1},
            {1, 0, 1},   {0, -1, -1}, {0, 1, -1},  {0, -1, 1},  {0, 1, 1},   {-1, -1, -1}, {1, -1, -1},
            {-1, 1, -1}, {1, 1, -1},  {-1, -1, 1}, {1, -1, 1},  {-1, 1, 1},  {1, 1, 1}};
#pragma unroll 1
        for (int u = 0; u < mode; ++u) {
            const int2 r = cell_lookup(g, cx + off[u][0], cy + off[u][1], cz + off[u][2]);
            if (r.y <= r.x) continue;
            const float4 b = __ldg(pts + r.x), m = __ldg(vmu + r.x);
            const float4 c0 = __ldg(vcov + 2 * (int64_t)r.x), c1 = __ldg(vcov + 2 * (int64_t)r.x + 1);
            const float cq[6] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y};
            // mean = first point + offset, exactly in fp64; d = mean - T p
            const float dx = (float)(((double)b.x + (double)m.x) - pp[0]);
            const float dy = (float)(((double)b.y + (double)m.y) - pp[1]);
            const float dz = (float)(((double)b.z + (double)m.z) - pp[2]);
            accumulate_terms<ERROR_ONLY, true>(P, pp, dx, dy, dz, cp, cq, acc, (double)m.w);
            cnt += 1.0;
        }
    }
    // warp tree -> fixed block tree -> block partials -> the last block's fixed-order pass
    __shared__ double sh[kVB / 32][kVNV];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int c = 0; c < 28; ++c) {
        if (ERROR_ONLY && c < 27) continue;
        const double v = vwarp_sum(acc[c]);
        if (lane == 0) sh[wid][c] = v;
    }
    {
        const double v = vwarp_sum(cnt);
        if (lane == 0) sh[wid][28] = v;
    }
    __syncthreads();
    if (threadIdx.x < kVNV) {
        const int c = threadIdx.x;
        double v = 0.0;
        if (!(ERROR_ONLY && c < 27)) {
#pragma unroll
            for (int w = 0; w < kVB / 32; ++w) v += sh[w][c];
        }
        partials[(int64_t)blockIdx.x * kVNV + c] = v;
    }
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = (atomicAdd(done, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!last) return;
    __threadfence();
    constexpr int kSub = 8;
    __shared__ double part[kSub][kVNV];
    const int nb = gridDim.x;
    if (threadIdx.x < kSub * kVNV) {
        const int c = threadIdx.x % kVNV, sub = threadIdx.x / kVNV;
        double v = 0.0;
        for (int b = sub; b < nb; b += kSub) v += __ldcg(partials + (int64_t)b * kVNV + c);
        part[sub][c] = v;
    }
    __syncthreads();
    if (threadIdx.x < kVNV) {
        double v = 0.0;
#pragma unroll
        for (int sub = 0; sub < kSub; ++sub) v += part[sub][threadIdx.x];
        out29[threadIdx.x] = v;
    }
    if (threadIdx.x == 0) *done = 0u;
}

__global__ void k_vzero29(double* out29) {
    if (threadIdx.x < 29) out29[threadIdx.x] = 0.0;
}

}  // namespace

int attach_voxels(gicp_index_s* idx, const float* cov, cudaStream_t s) {
    if (!idx->vox_mu) {
        if (cudaMallocAsync(&idx->vox_mu, idx->n * sizeof(float4), s) != cudaSuccess ||
            cudaMallocAsync(&idx->vox_cov, idx->n * 2 * sizeof(float4), s) != cudaSuccess) {
            cudaGetLastError();
            return set_error(GICP_ENOMEM, "voxel statistics allocation failed");
        }
        idx->device_bytes += idx->n * 3 * (int64_t)sizeof(float4);
    }
    const int64_t cap = idx->hash_cap[0];
    k_voxel_stats<<<(unsigned)((cap + 255) / 256), 256, 0, s>>>(idx->lv[0].hash, cap, idx->pts, cov, idx->vox_mu,
                                                                 idx->vox_cov);
    idx->vox_attached = cov;
    return check_cuda(cudaGetLastError(), "voxel statistics");
}

size_t vgicp_scratch_bytes(int64_t ns) { return (size_t)((ns + kVB - 1) / kVB) * kVNV * sizeof(double) + 256; }

int launch_linearize_vgicp(const float* src, const float* src_cov, int64_t ns, const gicp_index_s* tgt,
                           const double T[16], const double* pivot, int mode, int flags, int* base, double* out29,
                           cudaStream_t s, const LinScratch* pre) {
    if (ns == 0) {
        k_vzero29<<<1, 32, 0, s>>>(out29);
        return check_cuda(cudaGetLastError(), "vgicp launch");
    }
    const Pose P = make_pose(T, pivot);
    const int64_t nb = (ns + kVB - 1) / kVB;
    void* scratch = nullptr;
    unsigned* done;
    double* partials;
    if (pre) {
        done = pre->done;
        partials = pre->partials;
    } else {
        if (cudaMallocAsync(&scratch, vgicp_scratch_bytes(ns), s) != cudaSuccess) {
            cudaGetLastError();
            return set_error(GICP_ENOMEM, "vgicp scratch allocation failed");
        }
        done = (unsigned*)scratch;
        partials = (double*)((char*)scratch + 256);
        const int rc = check_cuda(cudaMemsetAsync(done, 0, sizeof(unsigned), s), "memset");
        if (rc) {
            cudaFreeAsync(scratch, s);
            return rc;
        }
    }
#define GICP_VG(E, R)                                                                                           \
    k_linearize_vgicp<E, R><<<(unsigned)nb, kVB, 0, s>>>(src, src_cov, ns, tgt->pts, tgt->lv[0], tgt->vox_mu,        \
                                                        tgt->vox_cov, P, mode, base, partials, done, out29)
    const bool eo = flags & GICP_LIN_ERROR_ONLY, re = flags & GICP_LIN_REUSE_CORR;
    if (eo && re)
        GICP_VG(true, true);
    else if (eo)
        GICP_VG(true, false);
    else if (re)
        GICP_VG(false, true);
    else
        GICP_VG(false, false);
#undef GICP_VG
    const int rc = check_cuda(cudaGetLastError(), "vgicp launch");
    if (scratch) cudaFreeAsync(scratch, s);
    return rc;
}

}  // namespace gicp
