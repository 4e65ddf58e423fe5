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

}  // namespace

int launch_covariances(const float* xyz, int64_t n, const int32_t* nbr, int64_t m, int k, float eps, float* cov,
                       cudaStream_t s) {
    if (m == 0) return GICP_OK;
    k_cov<<<(unsigned)((m + kBlock - 1) / kBlock), kBlock, 0, s>>>(xyz, n, nbr, m, k, eps, cov);
    return check_cuda(cudaGetLastError(), "covariances launch");
}

}  // namespace gicp
