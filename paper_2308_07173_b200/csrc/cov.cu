// cov.cu -- gicp_covariances: per-point GICP covariance from a given neighbour table.
//
// Paper: "computing covariance when estimate the C^p_i and C^q_i" (PAPER.md l.404,
// l.413, l.798). Definition: header gicp.h / DESIGN.md readings R6, R7, R11.
// One thread per row; the K neighbours are gathered twice (mean, then centred
// scatter) -- the second pass hits L1. The fused path in knn.cu avoids the
// nbr round trip through HBM altogether.
#include "cov_device.cuh"
#include "gicp_internal.cuh"

namespace gicp {
namespace {

constexpr int kBlock = 128;

__device__ __forceinline__ void load3(const float* __restrict__ xyz, int64_t n, int j, float& x, float& y, float& z) {
    j = min(max(j, 0), (int)(n - 1));
    x = __ldg(xyz + 3 * (int64_t)j);
    y = __ldg(xyz + 3 * (int64_t)j + 1);
    z = __ldg(xyz + 3 * (int64_t)j + 2);
}

__global__ void __launch_bounds__(kBlock) k_cov(const float* __restrict__ xyz, int64_t n,
                                                const int32_t* __restrict__ nbr, int64_t m, int K, float eps,
                                                float* __restrict__ cov) {
    const int64_t i = blockIdx.x * (int64_t)kBlock + threadIdx.x;
    if (i >= m) return;
    const int32_t* row = nbr + i * K;
    float x0, y0, z0;
    load3(xyz, n, __ldg(row), x0, y0, z0);
    float sx = 0.f, sy = 0.f, sz = 0.f;
    for (int r = 0; r < K; ++r) {
        float x, y, z;
        load3(xyz, n, __ldg(row + r), x, y, z);
        sx += x - x0;
        sy += y - y0;
        sz += z - z0;
    }
    const float invk = 1.0f / (float)K;
    const float mx = sx * invk, my = sy * invk, mz = sz * invk;
    float c00 = 0.f, c01 = 0.f, c02 = 0.f, c11 = 0.f, c12 = 0.f, c22 = 0.f;
    for (int r = 0; r < K; ++r) {
        float x, y, z;
        load3(xyz, n, __ldg(row + r), x, y, z);
        x = (x - x0) - mx;
        y = (y - y0) - my;
        z = (z - z0) - mz;
        c00 = fmaf(x, x, c00);
        c01 = fmaf(x, y, c01);
        c02 = fmaf(x, z, c02);
        c11 = fmaf(y, y, c11);
        c12 = fmaf(y, z, c12);
        c22 = fmaf(z, z, c22);
    }
    float c[6];
    plane_cov(c00 * invk, c01 * invk, c02 * invk, c11 * invk, c12 * invk, c22 * invk, eps, c);
    float2* o = reinterpret_cast<float2*>(cov + i * 6);
    o[0] = make_float2(c[0], c[1]);
    o[1] = make_float2(c[2], c[3]);
    o[2] = make_float2(c[4], c[5]);
}

// Kernel-descriptor weighted covariance (Table I l.420-435; SURVEY.md
// §8(f) #1; readings R19-R21): w_j = K(q - o, x_j - o) clamped at 0, all
// zero -> uniform; weighted mean / scatter (1 / sum w), then the chosen
// regularisation. Distance kernels are evaluated relative to the row's nearest
// candidate, w_j * exp(+K(d_min)) -- a constant factor per row, which cancels in
// the mean and the scatter and keeps fp32 exp from underflowing. Polynomial in
// fp64 (pow of large dot products).
__device__ __forceinline__ float kd_base(const CovKD& p, float d2, float d2min) {
    switch (p.kind) {
        case GICP_KD_RBF: return expf(-(d2 - d2min) * p.sigma);
        case GICP_KD_GAUSSIAN: return expf(-(d2 - d2min) / (2.0f * p.sigma * p.sigma));
        case GICP_KD_LAPLACIAN: return expf(-(sqrtf(d2) - sqrtf(d2min)) / p.sigma);
        default: return 1.0f;
    }
}

__global__ void __launch_bounds__(kBlock) k_cov_kd(const float* __restrict__ xyz, int64_t n,
                                                   const float* __restrict__ q, const int32_t* __restrict__ nbr,
                                                   int64_t m, int K, CovKD p, float* __restrict__ cov) {
    const int64_t i = blockIdx.x * (int64_t)kBlock + threadIdx.x;
    if (i >= m) return;
    const int32_t* row = nbr + i * K;
    const float* qi = q ? q + 3 * i : xyz + 3 * i;
    const float qx = qi[0], qy = qi[1], qz = qi[2];
    // kernel-space query (origin-relative; HI on the non-negative part)
    float ux = qx - p.ox, uy = qy - p.oy, uz = qz - p.oz;
    if (p.kind == GICP_KD_HI) {
        ux = fmaxf(ux, 0.f);
        uy = fmaxf(uy, 0.f);
        uz = fmaxf(uz, 0.f);
    }
    const bool dist_kernel = p.kind == GICP_KD_RBF || p.kind == GICP_KD_GAUSSIAN || p.kind == GICP_KD_LAPLACIAN;
    float d2min = 0.f;
    if (dist_kernel) {
        d2min = __int_as_float(0x7f800000);
        for (int r = 0; r < K; ++r) {
            float x, y, z;
            load3(xyz, n, __ldg(row + r), x, y, z);
            d2min = fminf(d2min, dist2(qx, qy, qz, x, y, z));
        }
    }
    auto weight = [&](float x, float y, float z) -> float {
        float w = 1.0f;
        if (dist_kernel) {
            w = kd_base(p, dist2(qx, qy, qz, x, y, z), d2min);
        } else if (p.kind == GICP_KD_POLYNOMIAL) {
            const double dot = (double)ux * (double)(x - p.ox) + (double)uy * (double)(y - p.oy) +
                               (double)uz * (double)(z - p.oz);
            const double b = (double)p.alpha * dot + (double)p.c;
            double v = 1.0;
            for (int e = 0; e < p.degree; ++e) v *= b;
            w = (float)v;
        } else if (p.kind == GICP_KD_HI) {
            const float vx = fmaxf(x - p.ox, 0.f), vy = fmaxf(y - p.oy, 0.f), vz = fmaxf(z - p.oz, 0.f);
            const float sx = ux + uy + uz;
            w = sx > 0.f ? (fminf(ux, vx) + fminf(uy, vy) + fminf(uz, vz)) / sx : 1.0f;
        }
        return (w > 0.0f && w <= 3.0e38f) ? w : 0.0f;  // clamp negatives (and NaN / inf) to 0
    };
    float x0, y0, z0;
    load3(xyz, n, __ldg(row), x0, y0, z0);
    float W = 0.f, sx = 0.f, sy = 0.f, sz = 0.f;
    for (int r = 0; r < K; ++r) {
        float x, y, z;
        load3(xyz, n, __ldg(row + r), x, y, z);
        const float w = weight(x, y, z);
        W += w;
        sx = fmaf(w, x - x0, sx);
        sy = fmaf(w, y - y0, sy);
        sz = fmaf(w, z - z0, sz);
    }
    const bool uniform = !(W > 0.f);
    if (uniform) {
        W = (float)K;
        sx = sy = sz = 0.f;
        for (int r = 0; r < K; ++r) {
            float x, y, z;
            load3(xyz, n, __ldg(row + r), x, y, z);
            sx += x - x0;
            sy += y - y0;
            sz += z - z0;
        }
    }
    const float invW = 1.0f / W;
    const float mx = sx * invW, my = sy * invW, mz = sz * invW;
    float c00 = 0.f, c01 = 0.f, c02 = 0.f, c11 = 0.f, c12 = 0.f, c22 = 0.f;
    for (int r = 0; r < K; ++r) {
        float x, y, z;
        load3(xyz, n, __ldg(row + r), x, y, z);
        const float w = uniform ? 1.0f : weight(x, y, z);
        x = (x - x0) - mx;
        y = (y - y0) - my;
        z = (z - z0) - mz;
        const float wx = w * x, wy = w * y;
        c00 = fmaf(wx, x, c00);
        c01 = fmaf(wx, y, c01);
        c02 = fmaf(wx, z, c02);
        c11 = fmaf(wy, y, c11);
        c12 = fmaf(wy, z, c12);
        c22 = fmaf(w * z, z, c22);
    }
    float c[6];
    if (p.reg == GICP_REG_PLANE)
        plane_cov(c00 * invW, c01 * invW, c02 * invW, c11 * invW, c12 * invW, c22 * invW, p.eps, c);
    else
        clamp_cov(c00 * invW, c01 * invW, c02 * invW, c11 * invW, c12 * invW, c22 * invW, p.reg, p.eps, c);
    float2* o = reinterpret_cast<float2*>(cov + i * 6);
    o[0] = make_float2(c[0], c[1]);
    o[1] = make_float2(c[2], c[3]);
    o[2] = make_float2(c[4], c[5]);
}

}  // namespace

int launch_covariances(const float* xyz, int64_t n, const int32_t* nbr, int64_t m, int k, float eps, float* cov,
                       cudaStream_t s) {
    if (m == 0) return GICP_OK;
    k_cov<<<(unsigned)((m + kBlock - 1) / kBlock), kBlock, 0, s>>>(xyz, n, nbr, m, k, eps, cov);
    return check_cuda(cudaGetLastError(), "covariances launch");
}

int launch_covariances_kd(const float* xyz, int64_t n, const float* q, const int32_t* nbr, int64_t m, int k,
                          const CovKD& p, float* cov, cudaStream_t s) {
    if (m == 0) return GICP_OK;
    k_cov_kd<<<(unsigned)((m + kBlock - 1) / kBlock), kBlock, 0, s>>>(xyz, n, q, nbr, m, k, p, cov);
    return check_cuda(cudaGetLastError(), "covariances launch");
}

}  // namespace gicp
