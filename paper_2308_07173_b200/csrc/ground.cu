// ground.cu -- z-vote ground filter ("project to the 2-D grid
// to vote the points corresponding to the grid-cell ... a hashing algorithm
// during the voting ... filter out ground points without matrix computation for
// plane extraction"; reading R24).
//
// cell (u, v) = (floor(fl32(x * fl32(1/cell))), floor(fl32(y * fl32(1/cell)))) in
// the points' frame; a point is a vertical feature (kept) iff its cell holds at
// least min_count points. Two passes over the points: vote into an open-
// addressing hash of the occupied cells (CAS on the key, atomicAdd on the
// count), then read each point's count back. Integer work on an fp32 decision
// taken exactly as the definition states: bit-exact.
#include "gicp_internal.cuh"

namespace gicp {
namespace {

struct VoteEntry {
    unsigned long long key;
    unsigned long long count;  // 64-bit slot keeps the entry 16-B aligned
};

__device__ __forceinline__ unsigned long long uv_key(float x, float y, float inv) {
    const float tu = __fmul_rn(x, inv), tv = __fmul_rn(y, inv);
    const double fu = floor((double)tu), fv = floor((double)tv);
    const long long u = (long long)fmin(fmax(fu, -2147483646.0), 2147483646.0);
    const long long v = (long long)fmin(fmax(fv, -2147483646.0), 2147483646.0);
    return ((unsigned long long)(u + 2147483648ll) << 32) | (unsigned long long)(v + 2147483648ll);
}

__device__ __forceinline__ unsigned long long vote_slot(unsigned long long key, int bits) {
    return (key * 0x9E3779B97F4A7C15ull) >> (64 - bits);
}

__global__ void k_vote_clear(VoteEntry* T, int64_t cap) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < cap) {
        T[i].key = kEmptyKey;
        T[i].count = 0ull;
    }
}

__global__ void k_vote(const float* __restrict__ xyz, int64_t n, float inv, VoteEntry* T, int bits) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const unsigned long long key = uv_key(xyz[3 * i], xyz[3 * i + 1], inv);
    const unsigned long long mask = (1ull << bits) - 1ull;
    unsigned long long h = vote_slot(key, bits);
    while (true) {
        const unsigned long long prev = atomicCAS(&T[h].key, kEmptyKey, key);
        if (prev == kEmptyKey || prev == key) {
            atomicAdd(&T[h].count, 1ull);
            return;
        }
        h = (h + 1) & mask;
    }
}

__global__ void k_vote_read(const float* __restrict__ xyz, int64_t n, float inv, const VoteEntry* __restrict__ T,
                            int bits, int min_count, uint8_t* __restrict__ keep, int32_t* __restrict__ count) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const unsigned long long key = uv_key(xyz[3 * i], xyz[3 * i + 1], inv);
    const unsigned long long mask = (1ull << bits) - 1ull;
    unsigned long long h = vote_slot(key, bits);
    while (__ldg(&T[h].key) != key) h = (h + 1) & mask;
    const unsigned long long c = __ldg(&T[h].count);
    keep[i] = c >= (unsigned long long)min_count;
    if (count) count[i] = (int32_t)c;
}

}  // namespace

int launch_ground_filter(const float* xyz, int64_t n, float cell, int min_count, uint8_t* keep, int32_t* count,
                         cudaStream_t s) {
    if (n == 0) return GICP_OK;
    int bits = 1;
    while ((1ll << bits) < 2 * n) ++bits;
    const int64_t cap = 1ll << bits;
    VoteEntry* T = nullptr;
    if (cudaMallocAsync((void**)&T, cap * sizeof(VoteEntry), s) != cudaSuccess) {
        cudaGetLastError();
        return set_error(GICP_ENOMEM, "ground filter: vote table allocation failed");
    }
    volatile float iv = 1.0f / cell;  // fl32(1/cell), as the definition
    const float inv = iv;
    k_vote_clear<<<(unsigned)((cap + 255) / 256), 256, 0, s>>>(T, cap);
    k_vote<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(xyz, n, inv, T, bits);
    k_vote_read<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(xyz, n, inv, T, bits, min_count, keep, count);
    const int rc = check_cuda(cudaGetLastError(), "ground filter");
    cudaFreeAsync(T, s);
    return rc;
}

}  // namespace gicp
