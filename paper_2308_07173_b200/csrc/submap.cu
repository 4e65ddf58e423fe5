// submap.cu -- sliding-window submap of a race-track map (PAPER.md l.477-481:
// "associate each pose on the race line with its corresponding point cloud map"
// with a GPU hash; "utilizing points from M_i^psi instead of processing the
// entire unified map"; R26).
//
// Every map point carries an arc-length bucket id (the caller's race-line
// parametrisation). Build: one stable radix sort of (bucket, index) and the
// bucket start table -- bucket ids are dense, so the table is a perfect hash
// from a race-line position to its map points. Query: the buckets center - r ..
// center + r of the closed track are at most two contiguous runs of the sorted
// order: one or two device-to-device copies.
#include <cub/cub.cuh>

#include <vector>

#include "gicp_internal.cuh"

struct gicp_submap_s {
    int64_t n = 0;
    int n_buckets = 0;
    int32_t* order = nullptr;          // point indices sorted by bucket (stable)
    std::vector<int64_t> starts;       // host copy of the bucket start table [n_buckets + 1]
    cudaStream_t stream = nullptr;
};

namespace gicp {
namespace {

__global__ void k_bucket_count(const int32_t* __restrict__ bucket, int64_t n, int nb, int* __restrict__ cnt,
                               int* __restrict__ bad, int32_t* __restrict__ keys, int32_t* __restrict__ vals) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int b = bucket[i];
    if (b < 0 || b >= nb) {
        atomicOr(bad, 1);
        keys[i] = 0;
    } else {
        atomicAdd(cnt + b, 1);
        keys[i] = b;
    }
    vals[i] = (int32_t)i;
}

}  // namespace
}  // namespace gicp

using namespace gicp;

GICP_API int gicp_submap_build(const int32_t* bucket, int64_t n, int n_buckets, gicp_submap* out, void* stream) {
    if (!out || n < 0 || (n > 0 && !bucket) || n_buckets < 1 || n >= (1ll << 31) - 1)
        return set_error(GICP_EINVAL, "gicp_submap_build: null / n / n_buckets");
    *out = nullptr;
    cudaStream_t s = (cudaStream_t)stream;
    gicp_submap sm = new gicp_submap_s;
    sm->n = n;
    sm->n_buckets = n_buckets;
    sm->stream = s;
    sm->starts.assign((size_t)n_buckets + 1, 0);
    if (n == 0) {
        *out = sm;
        return GICP_OK;
    }
    int bits = 1;
    while ((1ll << bits) < n_buckets) ++bits;
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, (int32_t*)nullptr, (int32_t*)nullptr, (int32_t*)nullptr,
                                    (int32_t*)nullptr, (int)n, 0, bits, s);
    char* buf = nullptr;
    const size_t bytes = (size_t)n * 12 + (size_t)(n_buckets + 2) * 4 + tb + 64;
    if (cudaMallocAsync((void**)&buf, bytes, s) != cudaSuccess ||
        cudaMallocAsync((void**)&sm->order, n * sizeof(int32_t), s) != cudaSuccess) {
        cudaGetLastError();
        if (buf) cudaFreeAsync(buf, s);
        delete sm;
        return set_error(GICP_ENOMEM, "gicp_submap_build: allocation failed");
    }
    int32_t* keys = (int32_t*)buf;
    int32_t* vals = keys + n;
    int32_t* kout = vals + n;
    int* cnt = (int*)(kout + n);
    int* bad = cnt + n_buckets;
    void* temp = (void*)(((uintptr_t)(bad + 1) + 15) & ~(uintptr_t)15);
    int rc = check_cuda(cudaMemsetAsync(cnt, 0, (n_buckets + 1) * sizeof(int), s), "memset");
    if (!rc) {
        k_bucket_count<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(bucket, n, n_buckets, cnt, bad, keys, vals);
        cub::DeviceRadixSort::SortPairs(temp, tb, keys, kout, vals, sm->order, (int)n, 0, bits, s);
        rc = check_cuda(cudaGetLastError(), "submap build");
    }
    std::vector<int> hc((size_t)n_buckets + 1, 0);
    if (!rc) rc = read_small(hc.data(), cnt, (n_buckets + 1) * sizeof(int), s);
    cudaFreeAsync(buf, s);
    if (!rc && hc[n_buckets]) rc = set_error(GICP_EINVAL, "gicp_submap_build: bucket id outside [0, n_buckets)");
    if (rc) {
        cudaFreeAsync(sm->order, s);
        delete sm;
        return rc;
    }
    for (int b = 0; b < n_buckets; ++b) sm->starts[b + 1] = sm->starts[b] + hc[b];
    *out = sm;
    return GICP_OK;
}

GICP_API void gicp_submap_free(gicp_submap sm) {
    if (!sm) return;
    if (sm->order) cudaFreeAsync(sm->order, sm->stream);
    delete sm;
}

GICP_API int gicp_submap_query(gicp_submap sm, int center, int radius, int32_t* out, int64_t* count, void* stream) {
    if (!sm || !count || radius < 0 || center < 0 || center >= sm->n_buckets)
        return set_error(GICP_EINVAL, "gicp_submap_query: null / center / radius");
    cudaStream_t s = (cudaStream_t)stream;
    const int nb = sm->n_buckets;
    const int64_t span = std::min<int64_t>(2 * (int64_t)radius + 1, nb);
    const int lo = (int)((((int64_t)center - radius) % nb + nb) % nb);
    const int64_t hi_excl = lo + span;  // in unwrapped bucket numbers
    auto run = [&](int64_t b0, int64_t b1, int64_t at) -> int64_t {  // buckets [b0, b1) of the sorted order
        const int64_t a = sm->starts[b0], b = sm->starts[b1];
        if (b > a && out)
            cudaMemcpyAsync(out + at, sm->order + a, (b - a) * sizeof(int32_t), cudaMemcpyDeviceToDevice, s);
        return b - a;
    };
    int64_t m = 0;
    if (hi_excl <= nb) {
        m = run(lo, hi_excl, 0);
    } else {
        m = run(lo, nb, 0);
        m += run(0, hi_excl - nb, m);
    }
    if (m > 0 && !out) return set_error(GICP_EINVAL, "gicp_submap_query: null out");
    *count = m;
    return check_cuda(cudaGetLastError(), "submap query");
}
