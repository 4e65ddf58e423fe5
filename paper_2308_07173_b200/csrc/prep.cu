// prep.cu -- data re-layout helpers of the linearisation path:
//  * attach_covariances: the target covariances permuted into the index's sorted
//    order as 2 x float4 per point (one 32-B sector), so a correspondence found
//    at sorted position j reads its covariance next to its coordinates;
//  * sort_source: gicp_align visits the source points in Morton order of their
//    own frame (a rigid motion preserves spatial coherence), so the 32 lanes of a
//    warp search the same part of the target grid.
#include <cub/cub.cuh>

#include "gicp_internal.cuh"

namespace gicp {
namespace {

__global__ void k_attach_cov(const float4* __restrict__ pts, const float* __restrict__ cov, int64_t n,
                             float4* __restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t o = __float_as_int(__ldg(pts + i).w);
    const float* c = cov + 6 * o;
    out[2 * i] = make_float4(c[0], c[1], c[2], c[3]);
    out[2 * i + 1] = make_float4(c[4], c[5], 0.f, 0.f);
}

__global__ void k_source_keys(const float* __restrict__ src, int64_t n, float inv, const int64_t* __restrict__ offs,
                              int nseg, unsigned long long* __restrict__ keys, int* __restrict__ vals) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    unsigned c[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        float t = src[3 * i + a] * inv;
        // 10 bits per axis around the frame origin (+-512 cells; the order only
        // serves locality, so clamping far points costs locality, never results)
        t = fminf(fmaxf(t, -512.0f), 511.0f);
        c[a] = (unsigned)((int)floorf(t) + 512);
    }
    unsigned long long seg = 0;
    if (offs) {  // batched: the registration of point i (largest s with offs[s] <= i) in the high bits
        int lo = 0, hi = nseg - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (offs[mid] <= i) lo = mid; else hi = mid - 1;
        }
        seg = (unsigned long long)lo << 30;
    }
    keys[i] = seg | cell_key((int)c[0], (int)c[1], (int)c[2]);
    vals[i] = (int)i;
}

__global__ void k_gather_source(const float* __restrict__ src, const float* __restrict__ cov,
                                const int* __restrict__ perm, int64_t n, float* __restrict__ src_p,
                                float* __restrict__ cov_p) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t j = perm[i];
#pragma unroll
    for (int a = 0; a < 3; ++a) src_p[3 * i + a] = src[3 * j + a];
#pragma unroll
    for (int a = 0; a < 6; ++a) cov_p[6 * i + a] = cov[6 * j + a];
}

}  // namespace

int attach_covariances(gicp_index_s* idx, const float* cov, cudaStream_t s) {
    if (!idx->cov_sorted) {
        if (cudaMallocAsync(&idx->cov_sorted, idx->n * 2 * sizeof(float4), s) != cudaSuccess) {
            cudaGetLastError();
            idx->cov_sorted = nullptr;
            return set_error(GICP_ENOMEM, "covariance attach: allocation failed");
        }
        idx->device_bytes += idx->n * 2 * (int64_t)sizeof(float4);
    }
    k_attach_cov<<<(unsigned)((idx->n + 255) / 256), 256, 0, s>>>(idx->pts, cov, idx->n, idx->cov_sorted);
    idx->cov_attached = cov;
    return check_cuda(cudaGetLastError(), "covariance attach");
}

int sort_source(const float* src, const float* src_cov, int64_t ns, float cell, float* src_p, float* cov_p,
                cudaStream_t s, const int64_t* offs, int nseg) {
    int segbits = 0;
    while (offs && (1 << segbits) < nseg) ++segbits;
    const int bits = 30 + segbits;
    void* buf = nullptr;
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, (unsigned long long*)nullptr, (unsigned long long*)nullptr,
                                    (int*)nullptr, (int*)nullptr, (int)ns, 0, bits, s);
    const size_t bytes = ns * (8 + 8 + 4 + 4) + tb + 64;
    if (cudaMallocAsync(&buf, bytes, s) != cudaSuccess) {
        cudaGetLastError();
        return set_error(GICP_ENOMEM, "source sort: allocation failed");
    }
    unsigned long long* k_in = (unsigned long long*)buf;
    unsigned long long* k_out = k_in + ns;
    int* v_in = (int*)(k_out + ns);
    int* v_out = v_in + ns;
    void* temp = (void*)(((uintptr_t)(v_out + ns) + 15) & ~(uintptr_t)15);
    const unsigned g = (unsigned)((ns + 255) / 256);
    k_source_keys<<<g, 256, 0, s>>>(src, ns, 1.0f / cell, offs, nseg, k_in, v_in);
    // stable: within a registration the order is the single-registration order
    cub::DeviceRadixSort::SortPairs(temp, tb, k_in, k_out, v_in, v_out, (int)ns, 0, bits, s);
    k_gather_source<<<g, 256, 0, s>>>(src, src_cov, v_out, ns, src_p, cov_p);
    const int rc = check_cuda(cudaGetLastError(), "source sort");
    cudaFreeAsync(buf, s);
    return rc;
}

}  // namespace gicp
