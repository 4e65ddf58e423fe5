// api.cu -- the extern "C" boundary of libgicp_b200 (declared in include/gicp.h):
// argument validation, thread-local errors, and the host LM loop of gicp_align.
#include <cuda_runtime.h>

#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>
#include <algorithm>

#include "gicp_internal.cuh"

#ifndef GICP_ALIGN_CACHE
#define GICP_ALIGN_CACHE 1  // gicp_align skips the search for certified correspondences (R27)
#endif


namespace gicp {

namespace {
thread_local std::string g_last_error;
}

int set_error(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

int check_cuda(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return GICP_OK;
    cudaGetLastError();
    return set_error(GICP_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

namespace {

// keep freed stream-ordered scratch in the pool (no OS round trips per call)
void init_pool_once() {
    static thread_local int dev_done = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev_done == dev) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    dev_done = dev;
}

bool finite_T(const double T[16]) {
    for (int i = 0; i < 16; ++i)
        if (!std::isfinite(T[i])) return false;
    return true;
}

// ---- host LM (gicp_align) ------------------------------------------------------
// SE(3) exponential for delta = (omega, v), T <- Exp(delta) T (left perturbation).
void se3_exp(const double d[6], double E[16]) {
    const double wx = d[0], wy = d[1], wz = d[2];
    const double W[9] = {0, -wz, wy, wz, 0, -wx, -wy, wx, 0};
    double W2[9];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) W2[3 * a + b] = W[3 * a] * W[b] + W[3 * a + 1] * W[3 + b] + W[3 * a + 2] * W[6 + b];
    const double th = std::sqrt(wx * wx + wy * wy + wz * wz);
    double A, B, C;
    bool small = th < 1e-10;
    if (small) {
        A = 1.0;
        B = 0.0;
        C = 0.0;
    } else {
        A = std::sin(th) / th;
        B = (1.0 - std::cos(th)) / (th * th);
        C = (th - std::sin(th)) / (th * th * th);
    }
    double Rm[9], V[9];
    for (int k = 0; k < 9; ++k) {
        const double I = (k % 4 == 0) ? 1.0 : 0.0;
        Rm[k] = small ? I + W[k] : I + A * W[k] + B * W2[k];
        V[k] = small ? I : I + B * W[k] + C * W2[k];
    }
    std::memset(E, 0, 16 * sizeof(double));
    for (int a = 0; a < 3; ++a) {
        for (int b = 0; b < 3; ++b) E[4 * a + b] = Rm[3 * a + b];
        E[4 * a + 3] = V[3 * a] * d[3] + V[3 * a + 1] * d[4] + V[3 * a + 2] * d[5];
    }
    E[15] = 1.0;
}

// Tr(c) Exp(delta) Tr(-c): the perturbation rotates about the pivot c
void pivoted_exp(const double d[6], const double c[3], double E[16]) {
    se3_exp(d, E);
    for (int a = 0; a < 3; ++a) E[4 * a + 3] += c[a] - (E[4 * a] * c[0] + E[4 * a + 1] * c[1] + E[4 * a + 2] * c[2]);
}

void mul44(const double A[16], const double B[16], double C[16]) {
    double t[16];
    for (int a = 0; a < 4; ++a)
        for (int b = 0; b < 4; ++b) {
            double s = 0.0;
            for (int k = 0; k < 4; ++k) s += A[4 * a + k] * B[4 * k + b];
            t[4 * a + b] = s;
        }
    std::memcpy(C, t, sizeof(t));
}

// (A) x = y, A 6x6 SPD, LDL^T without pivoting; false if not positive definite
bool ldlt6(const double A[36], const double y[6], double x[6]) {
    double L[6][6] = {}, D[6];
    for (int j = 0; j < 6; ++j) {
        double s = A[7 * j];
        for (int p = 0; p < j; ++p) s -= L[j][p] * L[j][p] * D[p];
        if (!(s > 0.0)) return false;
        D[j] = s;
        L[j][j] = 1.0;
        for (int i = j + 1; i < 6; ++i) {
            double t = A[6 * i + j];
            for (int p = 0; p < j; ++p) t -= L[i][p] * L[j][p] * D[p];
            L[i][j] = t / D[j];
        }
    }
    // L z = y, then D w = z, then L^T x = w
    double z[6];
    for (int i = 0; i < 6; ++i) {
        double s = y[i];
        for (int p = 0; p < i; ++p) s -= L[i][p] * z[p];
        z[i] = s;
    }
    for (int i = 0; i < 6; ++i) z[i] /= D[i];
    for (int i = 5; i >= 0; --i) {
        double s = z[i];
        for (int p = i + 1; p < 6; ++p) s -= L[p][i] * x[p];
        x[i] = s;
    }
    return true;
}

// Host-mapped result block of gicp_align (per host thread): the last block of a
// linearize launch writes out29 straight into it and then a sequence number to
// `flag`; the host spins on the flag instead of a D2H copy + stream sync.
struct MappedOut {
    double* h = nullptr;             // host view: 32 doubles, then the flag
    double* d = nullptr;             // device view of the same memory
    volatile unsigned* flag = nullptr;
    volatile unsigned* dflag = nullptr;
    unsigned seq = 0;
};
MappedOut* mapped_out() {
    static thread_local MappedOut m;
    if (!m.h) {
        void* p = nullptr;
        if (cudaHostAlloc(&p, 64 * sizeof(double), cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        void* dp = nullptr;
        if (cudaHostGetDevicePointer(&dp, p, 0) != cudaSuccess) {
            cudaGetLastError();
            cudaFreeHost(p);
            return nullptr;
        }
        std::memset(p, 0, 64 * sizeof(double));
        m.h = (double*)p;
        m.d = (double*)dp;
        m.flag = (volatile unsigned*)(m.h + 32);
        m.dflag = (volatile unsigned*)(m.d + 32);
    }
    return &m;
}

// wait for the launch that signals `seq`; polls the stream now and then so a
// failed launch is reported instead of spinning forever
int wait_mapped(MappedOut* m, unsigned seq, cudaStream_t s) {
    for (unsigned long it = 1;; ++it) {
        if (*m->flag == seq) {
            std::atomic_thread_fence(std::memory_order_acquire);
            return GICP_OK;
        }
        if ((it & 255) == 0) {
            const cudaError_t e = cudaStreamQuery(s);
            if (e == cudaSuccess) {
                if (*m->flag == seq) continue;
                return set_error(GICP_ECUDA, "gicp_align: linearize finished without its completion signal");
            }
            if (e != cudaErrorNotReady) return check_cuda(e, "gicp_align");
        }
    }
}

// opt-in per-launch device timing of gicp_align's linearisations (CUDA events on
// the launching stream): [0] speculative dual launches, [1] full linearisations,
// [2] trial costs. gicp_align_timing() enables / reads / resets it.
struct KernelTiming {
    static constexpr int kCap = 2048;  // launches timed per call (batched aligns: up to ~10 per iteration)
    int on = 0;
    cudaEvent_t e[2 * kCap] = {};
    int kind[kCap] = {};
    int64_t lpts[kCap] = {};  // source points the launch linearised (active registrations)
    int used = 0;  // event pairs recorded by the current call
    double ms[3] = {0, 0, 0};
    int64_t n[3] = {0, 0, 0};
    int64_t pts[3] = {0, 0, 0};
};
KernelTiming& kernel_timing() {
    static thread_local KernelTiming t;
    return t;
}
// read the recorded pairs (their stream has been synchronised) into the totals
void kernel_timing_collect(KernelTiming& t) {
    for (int i = 0; i < t.used; ++i) {
        float m = 0.f;
        if (cudaEventElapsedTime(&m, t.e[2 * i], t.e[2 * i + 1]) == cudaSuccess) {
            t.ms[t.kind[i]] += m;
            t.n[t.kind[i]] += 1;
            t.pts[t.kind[i]] += t.lpts[i];
        }
    }
    cudaGetLastError();
    t.used = 0;
}

struct Bytes256 {
    unsigned char b[256];
};

__global__ void k_export_bytes(const unsigned char* __restrict__ src, unsigned char* dst, size_t n) {
    for (size_t i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
    __threadfence_system();
}

__global__ void k_import_bytes(Bytes256 v, unsigned char* __restrict__ dst, size_t n) {
    for (size_t i = threadIdx.x; i < n; i += blockDim.x) dst[i] = v.b[i];
}

}  // namespace

int read_small(void* dst, const void* src_dev, size_t bytes, cudaStream_t s) {
    constexpr size_t kCap = 1 << 16;
    static thread_local unsigned char* h = nullptr;
    static thread_local unsigned char* d = nullptr;
    if (bytes > kCap) {  // large: a plain copy
        int rc = check_cuda(cudaMemcpyAsync(dst, src_dev, bytes, cudaMemcpyDeviceToHost, s), "D2H");
        return rc ? rc : check_cuda(cudaStreamSynchronize(s), "D2H sync");
    }
    if (!h) {
        void* p = nullptr;
        void* dp = nullptr;
        if (cudaHostAlloc(&p, kCap, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess ||
            cudaHostGetDevicePointer(&dp, p, 0) != cudaSuccess) {
            cudaGetLastError();
            if (p) cudaFreeHost(p);
            return set_error(GICP_ENOMEM, "host-mapped staging buffer");
        }
        h = (unsigned char*)p;
        d = (unsigned char*)dp;
    }
    if (bytes == 0) return GICP_OK;
    k_export_bytes<<<1, 256, 0, s>>>((const unsigned char*)src_dev, d, bytes);
    int rc = check_cuda(cudaGetLastError(), "small read");
    if (!rc) rc = check_cuda(cudaStreamSynchronize(s), "small read");
    if (!rc) std::memcpy(dst, h, bytes);
    return rc;
}

int write_small(void* dst_dev, const void* src, size_t bytes, cudaStream_t s) {
    if (bytes > sizeof(Bytes256)) return check_cuda(cudaMemcpyAsync(dst_dev, src, bytes, cudaMemcpyHostToDevice, s), "H2D");
    Bytes256 v;
    std::memcpy(v.b, src, bytes);
    k_import_bytes<<<1, 256, 0, s>>>(v, (unsigned char*)dst_dev, bytes);
    return check_cuda(cudaGetLastError(), "small write");
}

}  // namespace gicp

using namespace gicp;

GICP_API const char* gicp_last_error(void) { return g_last_error.c_str(); }

GICP_API int gicp_version(void) { return 100; }

GICP_API int gicp_build_index(const float* xyz, int64_t n, float cell_size, void* stream, gicp_index* out) {
    if (!xyz || !out) return set_error(GICP_EINVAL, "gicp_build_index: null pointer");
    if (n <= 0 || n >= (1ll << 31) - 1) return set_error(GICP_EINVAL, "gicp_build_index: n must be in [1, 2^31-1)");
    if (!std::isfinite(cell_size) || cell_size < 0.0f)
        return set_error(GICP_EINVAL, "gicp_build_index: cell_size must be finite and >= 0");
    init_pool_once();
    *out = nullptr;
    return build_index(xyz, n, cell_size, (cudaStream_t)stream, out);
}

GICP_API void gicp_index_free(gicp_index idx) {
    if (!idx) return;
    // stream-ordered release on the build stream (work queued after the build on
    // other streams must have completed: the caller's contract, as for cudaFree)
    cudaStream_t s = idx->stream;
    if (cudaFreeAsync(idx->pts, s) != cudaSuccess) {
        cudaGetLastError();
        s = nullptr;  // the build stream is gone: use the legacy stream
        cudaFreeAsync(idx->pts, s);
    }
    cudaFreeAsync(idx->pts_orig, s);
    cudaFreeAsync(idx->hash_mem, s);
    if (idx->cov_sorted) cudaFreeAsync(idx->cov_sorted, s);
    if (idx->adj_oc) cudaFreeAsync(idx->adj_oc, s);
    if (idx->adj_rng) cudaFreeAsync(idx->adj_rng, s);
    if (idx->adj_oc1) cudaFreeAsync(idx->adj_oc1, s);
    if (idx->vox_mu) cudaFreeAsync(idx->vox_mu, s);
    if (idx->vox_cov) cudaFreeAsync(idx->vox_cov, s);
    if (idx->adj_rng1) cudaFreeAsync(idx->adj_rng1, s);
    if (idx->tiles1) cudaFreeAsync(idx->tiles1, s);
    if (idx->tile_of) cudaFreeAsync(idx->tile_of, s);
    cudaGetLastError();
    delete idx;
}

static int check_k(int k, int64_t n, const char* fn);

// ---- index export / import (C5 sharding: one rank builds, the others receive) -----------
namespace {
struct IndexHeader {
    unsigned magic;
    int n_levels;
    int64_t n, n_cells, n_tiles1;
    int64_t hash_cap[kMaxLevels];
    int64_t adj_cap[2];
    Grid lv[kMaxLevels];  // hash pointers stored as slot offsets into hash_mem
    int64_t bytes[GICP_INDEX_MAX_BUFFERS];
};
static_assert(sizeof(IndexHeader) <= GICP_INDEX_HEADER_BYTES, "index header");
constexpr unsigned kIndexMagic = 0x47494350u;  // "GICP"
}  // namespace

GICP_API int gicp_index_export(gicp_index idx, void* header, void** buffers, int64_t* bytes, int* n_buffers) {
    if (!idx || !header || !buffers || !bytes || !n_buffers) return set_error(GICP_EINVAL, "gicp_index_export: null pointer");
    IndexHeader h{};
    h.magic = kIndexMagic;
    h.n_levels = idx->n_levels;
    h.n = idx->n;
    h.n_cells = idx->n_cells;
    h.n_tiles1 = idx->tiles1 ? idx->n_tiles1 : -1;
    int64_t total = 0;
    for (int l = 0; l < kMaxLevels; ++l) {
        h.hash_cap[l] = idx->hash_cap[l];
        h.lv[l] = idx->lv[l];
        h.lv[l].hash = (const HashEntry*)(intptr_t)(l < idx->n_levels ? idx->lv[l].hash - idx->hash_mem : 0);
        if (l < idx->n_levels) total += idx->hash_cap[l];
    }
    h.adj_cap[0] = idx->adj_rng ? idx->adj_cap[0] : 0;
    h.adj_cap[1] = idx->adj_rng1 ? idx->adj_cap[1] : 0;
    void* b[GICP_INDEX_MAX_BUFFERS] = {idx->pts, idx->pts_orig, idx->hash_mem, idx->adj_oc, idx->adj_rng, idx->adj_oc1,
                                       idx->adj_rng1, idx->tiles1, idx->tile_of};
    const int64_t n = idx->n;
    const int64_t sz[GICP_INDEX_MAX_BUFFERS] = {
        n * 16, n * 16, total * (int64_t)sizeof(HashEntry), idx->adj_oc ? n * 8 : 0, h.adj_cap[0] * 8,
        idx->adj_oc1 ? n * 8 : 0, h.adj_cap[1] * 8, idx->tiles1 ? (idx->n_tiles1 + 1) * 4 : 0,
        idx->tile_of ? n * 4 : 0};
    const int nb = 9;
    for (int i = 0; i < nb; ++i) {
        buffers[i] = sz[i] ? b[i] : nullptr;
        bytes[i] = sz[i];
        h.bytes[i] = sz[i];
    }
    *n_buffers = nb;
    std::memset(header, 0, GICP_INDEX_HEADER_BYTES);
    std::memcpy(header, &h, sizeof(h));
    return GICP_OK;
}

GICP_API int gicp_index_import(const void* header, const void* const* buffers, void* stream, gicp_index* out) {
    if (!header || !buffers || !out) return set_error(GICP_EINVAL, "gicp_index_import: null pointer");
    IndexHeader h;
    std::memcpy(&h, header, sizeof(h));
    if (h.magic != kIndexMagic || h.n_levels < 1 || h.n_levels > kMaxLevels || h.n <= 0)
        return set_error(GICP_EINVAL, "gicp_index_import: not an index header");
    init_pool_once();
    cudaStream_t s = (cudaStream_t)stream;
    gicp_index_s* idx = new gicp_index_s();
    idx->n = h.n;
    idx->n_cells = h.n_cells;
    idx->n_levels = h.n_levels;
    idx->stream = s;
    cudaGetDevice(&idx->device);
    void** dst[9] = {(void**)&idx->pts, (void**)&idx->pts_orig, (void**)&idx->hash_mem, (void**)&idx->adj_oc,
                     (void**)&idx->adj_rng, (void**)&idx->adj_oc1, (void**)&idx->adj_rng1, (void**)&idx->tiles1,
                     (void**)&idx->tile_of};
    for (int i = 0; i < 9; ++i) {
        if (!h.bytes[i]) continue;
        if (!buffers[i]) {
            gicp_index_free(idx);
            return set_error(GICP_EINVAL, "gicp_index_import: missing buffer");
        }
        if (cudaMallocAsync(dst[i], h.bytes[i], s) != cudaSuccess ||
            cudaMemcpyAsync(*dst[i], buffers[i], h.bytes[i], cudaMemcpyDeviceToDevice, s) != cudaSuccess) {
            cudaGetLastError();
            gicp_index_free(idx);
            return set_error(GICP_ENOMEM, "gicp_index_import: allocation / copy failed");
        }
        idx->device_bytes += h.bytes[i];
    }
    for (int l = 0; l < kMaxLevels; ++l) {
        idx->hash_cap[l] = h.hash_cap[l];
        idx->lv[l] = h.lv[l];
        idx->lv[l].hash = l < h.n_levels ? idx->hash_mem + (intptr_t)h.lv[l].hash : nullptr;
    }
    idx->adj_cap[0] = h.adj_cap[0];
    idx->adj_cap[1] = h.adj_cap[1];
    idx->n_tiles1 = h.n_tiles1 >= 0 ? h.n_tiles1 : 0;
    int rc = check_cuda(cudaStreamSynchronize(s), "gicp_index_import");
    if (rc) {
        gicp_index_free(idx);
        return rc;
    }
    *out = idx;
    return GICP_OK;
}

GICP_API int gicp_knn_query_order(gicp_index idx, const float* q, int64_t m, int32_t* perm, void* stream) {
    if (!idx) return set_error(GICP_EINVAL, "gicp_knn_query_order: null index");
    if (m < 0 || m >= (1ll << 31) - 1) return set_error(GICP_EINVAL, "gicp_knn_query_order: m out of range");
    if (m == 0) return GICP_OK;
    if (!q || !perm) return set_error(GICP_EINVAL, "gicp_knn_query_order: null pointer");
    init_pool_once();
    return launch_query_order(idx, q, m, perm, (cudaStream_t)stream);
}

GICP_API int gicp_knn_subset(gicp_index idx, const float* q, int64_t m, const int32_t* ids, int64_t n_ids, int k,
                             int32_t* nbr, float* d2, void* stream) {
    if (!idx) return set_error(GICP_EINVAL, "gicp_knn_subset: null index");
    if (m < 0 || m >= (1ll << 31) - 1 || n_ids < 0 || n_ids > m)
        return set_error(GICP_EINVAL, "gicp_knn_subset: m / n_ids out of range");
    int rc = check_k(k, idx->n, "gicp_knn_subset");
    if (rc) return rc;
    if (n_ids == 0) return GICP_OK;
    if (!q || !ids || !nbr || !d2) return set_error(GICP_EINVAL, "gicp_knn_subset: null pointer");
    init_pool_once();
    return launch_knn_subset(idx, q, ids, n_ids, k, nbr, d2, (cudaStream_t)stream);
}

GICP_API int gicp_index_attach_cov(gicp_index idx, const float* cov, void* stream) {
    if (!idx || !cov) return set_error(GICP_EINVAL, "gicp_index_attach_cov: null pointer");
    init_pool_once();
    return attach_covariances(idx, cov, (cudaStream_t)stream);
}

GICP_API int gicp_get_index_info(gicp_index idx, gicp_index_info* info) {
    if (!idx || !info) return set_error(GICP_EINVAL, "gicp_get_index_info: null pointer");
    info->n = idx->n;
    info->n_cells = idx->n_cells;
    info->cell_size = idx->lv[0].cell;
    info->origin[0] = idx->lv[0].ox;
    info->origin[1] = idx->lv[0].oy;
    info->origin[2] = idx->lv[0].oz;
    info->dims[0] = idx->lv[0].nx;
    info->dims[1] = idx->lv[0].ny;
    info->dims[2] = idx->lv[0].nz;
    info->n_levels = idx->n_levels;
    info->device_bytes = idx->device_bytes;
    return GICP_OK;
}

static int check_k(int k, int64_t n, const char* fn) {
    if (k < 1 || k > GICP_KMAX || k > n)
        return set_error(GICP_EK, std::string(fn) + ": k must satisfy 1 <= k <= min(32, n)");
    return GICP_OK;
}

GICP_API int gicp_knn(gicp_index idx, const float* q, int64_t m, int k, int32_t* nbr, float* d2, void* stream) {
    if (!idx) return set_error(GICP_EINVAL, "gicp_knn: null index");
    if (m < 0 || m >= (1ll << 31) - 1) return set_error(GICP_EINVAL, "gicp_knn: m out of range");
    int rc = check_k(k, idx->n, "gicp_knn");
    if (rc) return rc;
    if (m == 0) return GICP_OK;
    if (!q || !nbr || !d2) return set_error(GICP_EINVAL, "gicp_knn: null pointer");
    init_pool_once();
    return launch_knn(idx, q, m, k, nbr, d2, (cudaStream_t)stream);
}

GICP_API int gicp_knn_self(gicp_index idx, int k, int32_t* nbr, float* d2, void* stream) {
    if (!idx || !nbr || !d2) return set_error(GICP_EINVAL, "gicp_knn_self: null pointer");
    int rc = check_k(k, idx->n, "gicp_knn_self");
    if (rc) return rc;
    init_pool_once();
    return launch_knn_self(idx, k, 0.0f, nbr, d2, nullptr, (cudaStream_t)stream);
}

GICP_API int gicp_covariances(const float* xyz, int64_t n, const int32_t* nbr, int64_t m, int k, float eps,
                              float* cov, void* stream) {
    if (n <= 0 || m < 0) return set_error(GICP_EINVAL, "gicp_covariances: n must be > 0 and m >= 0");
    int rc = check_k(k, n, "gicp_covariances");
    if (rc) return rc;
    if (!(eps > 0.0f && eps <= 1.0f)) return set_error(GICP_EINVAL, "gicp_covariances: eps must be in (0, 1]");
    if (m == 0) return GICP_OK;
    if (!xyz || !nbr || !cov) return set_error(GICP_EINVAL, "gicp_covariances: null pointer");
    return launch_covariances(xyz, n, nbr, m, k, eps, cov, (cudaStream_t)stream);
}

GICP_API int gicp_covariances_kd(const float* xyz, int64_t n, const float* q, const int32_t* nbr, int64_t m, int k,
                                 const gicp_cov_params* p, float* cov, void* stream) {
    if (!p) return set_error(GICP_EINVAL, "gicp_covariances_kd: null params");
    if (n <= 0 || m < 0) return set_error(GICP_EINVAL, "gicp_covariances_kd: n must be > 0 and m >= 0");
    if (!q && m > n) return set_error(GICP_EINVAL, "gicp_covariances_kd: m > n without queries");
    int rc = check_k(k, n, "gicp_covariances_kd");
    if (rc) return rc;
    if (p->kernel < GICP_KD_UNIFORM || p->kernel > GICP_KD_LAPLACIAN)
        return set_error(GICP_EINVAL, "gicp_covariances_kd: unknown kernel");
    if (p->reg < GICP_REG_PLANE || p->reg > GICP_REG_NORMALIZED_MIN_EIG)
        return set_error(GICP_EINVAL, "gicp_covariances_kd: unknown regularisation");
    if (!(p->eps > 0.0f && p->eps <= 1.0f)) return set_error(GICP_EINVAL, "gicp_covariances_kd: eps must be in (0, 1]");
    const bool dist = p->kernel == GICP_KD_RBF || p->kernel == GICP_KD_GAUSSIAN || p->kernel == GICP_KD_LAPLACIAN;
    if (dist && !(p->sigma > 0.0f && std::isfinite(p->sigma)))
        return set_error(GICP_EINVAL, "gicp_covariances_kd: sigma must be finite and > 0");
    if (p->kernel == GICP_KD_POLYNOMIAL && (p->degree < 1 || p->degree > 16 || !std::isfinite(p->alpha) ||
                                            !std::isfinite(p->c)))
        return set_error(GICP_EINVAL, "gicp_covariances_kd: polynomial degree 1..16, finite alpha / c");
    if (!(std::isfinite(p->origin[0]) && std::isfinite(p->origin[1]) && std::isfinite(p->origin[2])))
        return set_error(GICP_EINVAL, "gicp_covariances_kd: non-finite origin");
    if (m == 0) return GICP_OK;
    if (!xyz || !nbr || !cov) return set_error(GICP_EINVAL, "gicp_covariances_kd: null pointer");
    const CovKD kd{p->kernel, p->sigma, p->alpha, p->c, p->degree, p->origin[0], p->origin[1], p->origin[2], p->reg,
                   p->eps};
    return launch_covariances_kd(xyz, n, q, nbr, m, k, kd, cov, (cudaStream_t)stream);
}

GICP_API int gicp_knn_cov_self(gicp_index idx, int k, float eps, int32_t* nbr, float* d2, float* cov, void* stream) {
    if (!idx || !cov) return set_error(GICP_EINVAL, "gicp_knn_cov_self: null pointer");
    int rc = check_k(k, idx->n, "gicp_knn_cov_self");
    if (rc) return rc;
    if (!(eps > 0.0f && eps <= 1.0f)) return set_error(GICP_EINVAL, "gicp_knn_cov_self: eps must be in (0, 1]");
    init_pool_once();
    return launch_knn_self(idx, k, eps, nbr, d2, cov, (cudaStream_t)stream);
}

GICP_API int gicp_linearize(const float* src, const float* src_cov, int64_t ns, gicp_index tgt, const float* tgt_cov,
                            const double T[16], const double* pivot, float max_corr_dist, int flags, double* out29,
                            int32_t* corr, void* stream) {
    if (!tgt || !tgt_cov || !T || !out29) return set_error(GICP_EINVAL, "gicp_linearize: null pointer");
    if (ns < 0 || ns >= (1ll << 31) - 1) return set_error(GICP_EINVAL, "gicp_linearize: ns out of range");
    if (ns > 0 && (!src || !src_cov)) return set_error(GICP_EINVAL, "gicp_linearize: null source");
    if (!(max_corr_dist > 0.0f) || !std::isfinite(max_corr_dist))
        return set_error(GICP_EINVAL, "gicp_linearize: max_corr_dist must be finite and > 0");
    if ((flags & GICP_LIN_REUSE_CORR) && !corr && ns > 0)
        return set_error(GICP_EINVAL, "gicp_linearize: REUSE_CORR needs corr");
    if (flags & ~(GICP_LIN_REUSE_CORR | GICP_LIN_ERROR_ONLY)) return set_error(GICP_EINVAL, "gicp_linearize: flags");
    if (!finite_T(T)) return set_error(GICP_EINVAL, "gicp_linearize: non-finite T");
    init_pool_once();
    if (pivot && !(std::isfinite(pivot[0]) && std::isfinite(pivot[1]) && std::isfinite(pivot[2])))
        return set_error(GICP_EINVAL, "gicp_linearize: non-finite pivot");
    return launch_linearize(src, src_cov, ns, tgt, tgt_cov, T, pivot, max_corr_dist, flags, out29, corr,
                            (cudaStream_t)stream);
}

// cube-stage level of the search (kLinCoarse): level 1 while the
// last pose step moved the source points by more than 0.8 level-0 cells (far-off
// poses: many nearest neighbours lie beyond level 0's cube), level 0 near the
// optimum. Exact either way; the choice only moves work (C3 sweep, DESIGN.md §4.3:
// 0.8 cell = 0.4 m was the fastest of 0.02 ... 1 m and never/always).
static double coarse_threshold(const gicp_index_s* tgt) {
    if (const char* e = getenv("GICP_LIN_COARSE_THR")) return atof(e);  // experiments
    return 0.8 * (double)tgt->lv[0].cell;
}
// the split evaluation's queue (linearize.cu: certificates, dense searches, terms)
// for the certificate paths; GICP_LIN_SPLIT=0 (build flag) keeps every launch fused
#ifndef GICP_LIN_SPLIT
#define GICP_LIN_SPLIT 1
#endif
static bool split_eval(int64_t n) { return GICP_LIN_SPLIT && n < (1ll << 30); }
// the batched align's deferred reduction (linearize.cu k_lin_reduce): the kernels skip
// the per-block fence + ticket; GICP_LIN_INLINE_REDUCE (env) keeps the in-kernel one
static bool deferred_reduce() {
    static const bool inl = getenv("GICP_LIN_INLINE_REDUCE") != nullptr;
    return !inl;
}
// |dv| + |dw| * 20 m (a typical range of the scan points): the step's point motion
static double step_displacement(const double* d) {
    return std::sqrt(d[3] * d[3] + d[4] * d[4] + d[5] * d[5]) + 20.0 * std::sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
}

GICP_API int gicp_align(const float* src, const float* src_cov, int64_t ns, gicp_index tgt, const float* tgt_cov,
                        const double T0[16], const gicp_align_params* prm, gicp_align_result* res, void* stream) {
    if (!tgt || !tgt_cov || !T0 || !prm || !res || (ns > 0 && (!src || !src_cov)))
        return set_error(GICP_EINVAL, "gicp_align: null pointer");
    if (ns < 0) return set_error(GICP_EINVAL, "gicp_align: ns < 0");
    if (ns < 6) return set_error(GICP_EDEGENERATE, "gicp_align: fewer than 6 source points");
    if (prm->max_iter < 1) return set_error(GICP_EINVAL, "gicp_align: max_iter < 1");
    if (!finite_T(T0)) return set_error(GICP_EINVAL, "gicp_align: non-finite T0");
    init_pool_once();
    cudaStream_t s = (cudaStream_t)stream;
    MappedOut* mo = mapped_out();
    if (!mo) return set_error(GICP_ENOMEM, "gicp_align: host-mapped buffer");
    const double* h = mo->h;
    // one scratch block for the whole alignment: out (31 doubles) | done counter |
    // block partials | two correspondence buffers | Morton-sorted copies of the
    // source and its covariances
    const int64_t nsa = ns > 0 ? ns : 1;
    const size_t lin_bytes = linearize_scratch_bytes(nsa);
    const size_t bytes = 512 + lin_bytes + 2 * nsa * sizeof(int32_t) + nsa * 9 * sizeof(float) + 256 +
                         (GICP_ALIGN_CACHE ? 4 * nsa * sizeof(float4) + 64 : 0);
    char* scratch = nullptr;
    if (cudaMallocAsync((void**)&scratch, bytes, s) != cudaSuccess) {
        cudaGetLastError();
        return set_error(GICP_ENOMEM, "gicp_align: scratch allocation failed");
    }
    LinScratch ls;
    ls.done = (unsigned*)(scratch + 256);
    ls.partials = (double*)(scratch + 512);
    int32_t* corr_a = (int32_t*)(scratch + 512 + lin_bytes);
    int32_t* corr_b = corr_a + nsa;
    float* src_p = (float*)(((uintptr_t)(corr_b + nsa) + 15) & ~(uintptr_t)15);
    float* cov_p = (float*)(((uintptr_t)(src_p + 3 * nsa) + 15) & ~(uintptr_t)15);  // float2 loads
    // the correspondence certificates paired with corr_a / corr_b (reading R27)
    float4* cache_a = nullptr;
    float4* cache_b = nullptr;
    // GICP_ALIGN_NOCACHE: always search (the bitwise A/B check in tests/test_gpu_parity.py)
    if (GICP_ALIGN_CACHE && getenv("GICP_ALIGN_NOCACHE") == nullptr) {
        cache_a = (float4*)(((uintptr_t)(cov_p + 6 * nsa) + 15) & ~(uintptr_t)15);
        cache_b = cache_a + nsa;
        if (split_eval(nsa)) {  // the split evaluation's search queue and counter
            ls.queue = cache_b + nsa;
            ls.queue2 = ls.queue + nsa;
            ls.qcount = (unsigned*)(ls.queue2 + nsa);
        }
    }
    auto cache_of = [&](const int32_t* c) -> float4* { return c == corr_a ? cache_a : (c == corr_b ? cache_b : nullptr); };
    int rc0 = check_cuda(cudaMemsetAsync(ls.done, 0, sizeof(unsigned), s), "memset");
    if (!rc0 && ns > 0) rc0 = sort_source(src, src_cov, ns, tgt->lv[0].cell, src_p, cov_p, s);
    if (rc0) {
        cudaFreeAsync(scratch, s);
        return rc0;
    }
    // one launch + one sync per evaluation: `old` != nullptr also evaluates the
    // trial cost with the previous correspondences (values 29, 30)
    ls.flag = mo->dflag;
    KernelTiming& kt = kernel_timing();
    const bool host_trace = getenv("GICP_DEBUG_ALIGN_HOST") != nullptr;  // diagnostics: host-side phases
    auto last_done = std::chrono::steady_clock::now();
    const double coarse_thr = coarse_threshold(tgt);
    double step_disp = INFINITY;  // the first linearisation: the initial guess's error is unknown
    auto go = [&](const double* T, const double* piv, int flags, int32_t* corr, const int32_t* old) -> int {
        ls.seq = ++mo->seq;
        if (step_disp > coarse_thr) flags |= kLinCoarse;
        ls.cache_new = (flags & GICP_LIN_REUSE_CORR) ? nullptr : cache_of(corr);
        ls.cache_old = old ? cache_of(old) : nullptr;
        // per-launch device time of the linearisations (bench.py's roofline): event
        // pairs on the stream, read once the alignment has finished
        const bool timed = kt.on && kt.used < KernelTiming::kCap;
        if (timed) cudaEventRecord(kt.e[2 * kt.used], s);
        const auto h0 = std::chrono::steady_clock::now();
        int rc = launch_linearize(src_p, cov_p, ns, tgt, tgt_cov, T, piv, prm->max_corr_dist, flags, mo->d,
                                  corr, s, &ls, old);
        const auto h1 = std::chrono::steady_clock::now();
        if (timed) {
            cudaEventRecord(kt.e[2 * kt.used + 1], s);
            kt.lpts[kt.used] = ns;
            kt.kind[kt.used++] = (old != nullptr) ? 0 : ((flags & GICP_LIN_ERROR_ONLY) ? 2 : 1);
        }
        if (!rc) rc = wait_mapped(mo, ls.seq, s);
        if (host_trace) {
            const auto h2 = std::chrono::steady_clock::now();
            auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
            fprintf(stderr, "[gicp align host] gap %.1f launch %.1f wait %.1f us\n", us(last_done, h0), us(h0, h1),
                    us(h1, h2));
            last_done = h2;
        }
        return rc;
    };
    auto lin = [&](const double* T, const double* piv, int32_t* corr, const int32_t* old) -> int {
        return go(T, piv, kLinCorrSpos, corr, old);
    };
    const bool debug = getenv("GICP_DEBUG_ALIGN") != nullptr;
    std::vector<float4> dbg_prev;
    double T[16];
    std::memcpy(T, T0, sizeof(T));
    double lambda = -1.0, nu = 2.0, err = 0.0;
    int converged = 0, it = 0, rc = GICP_OK;
    int64_t inl = 0;
    // pivot: the source frame origin in the target frame (the sensor position)
    double piv[3] = {T[3], T[7], T[11]};
    double lin29[29];  // the linearisation at the current T (about piv), corr in corr_a
    if ((rc = lin(T, piv, corr_a, nullptr)) == GICP_OK) std::memcpy(lin29, h, sizeof(lin29));
    for (it = 1; rc == GICP_OK && it <= prm->max_iter; ++it) {
        inl = (int64_t)lin29[28];
        if (inl < 6) {
            rc = set_error(GICP_EDEGENERATE, "gicp_align: fewer than 6 correspondences");
            break;
        }
        double Hm[36], b[6], delta[6] = {0, 0, 0, 0, 0, 0};
        for (int a = 0, o = 0; a < 6; ++a)
            for (int c = a; c < 6; ++c, ++o) Hm[6 * a + c] = Hm[6 * c + a] = lin29[o];
        for (int a = 0; a < 6; ++a) b[a] = lin29[21 + a];
        const double e = lin29[27];
        err = e;
        if (debug) {
            fprintf(stderr, "[gicp align] lin29 it=%d piv=(%.6f %.6f %.6f):", it, piv[0], piv[1], piv[2]);
            for (int c = 0; c < 29; ++c) fprintf(stderr, " %.9g", lin29[c]);
            fprintf(stderr, "\n");
        }
        bool done_now = false;
        if (!prm->lm) {
            double nb[6];
            for (int a = 0; a < 6; ++a) nb[a] = -b[a];
            if (!ldlt6(Hm, nb, delta)) {
                rc = set_error(GICP_EDEGENERATE, "gicp_align: singular H");
                break;
            }
            double E[16];
            pivoted_exp(delta, piv, E);
            mul44(E, T, T);
            step_disp = step_displacement(delta);
        } else {
            if (lambda < 0) {
                double mx = 0.0;
                for (int a = 0; a < 6; ++a) mx = std::fmax(mx, Hm[7 * a]);
                lambda = 1e-9 * mx;
            }
            bool accepted = false;
            for (int inner = 0; inner < 10; ++inner) {
                double Hl[36], nb[6];
                std::memcpy(Hl, Hm, sizeof(Hl));
                for (int a = 0; a < 6; ++a) {
                    Hl[7 * a] += lambda;
                    nb[a] = -b[a];
                }
                if (!ldlt6(Hl, nb, delta)) {
                    lambda *= nu;
                    nu *= 2.0;
                    continue;
                }
                double E[16], Tn[16];
                pivoted_exp(delta, piv, E);
                mul44(E, T, Tn);
                step_disp = step_displacement(delta);
                // trial: e' with the current correspondences at Tn. The first trial of
                // an iteration is usually accepted, so it also computes, speculatively,
                // the full linearisation at Tn in the same pass; later trials (after a
                // rejection) evaluate e' alone and linearise only once accepted.
                const double pn[3] = {Tn[3], Tn[7], Tn[11]};
                const bool spec = inner == 0;
                if (spec) {
                    if ((rc = lin(Tn, pn, corr_b, corr_a))) break;
                } else {
                    if ((rc = go(Tn, pn, kLinCorrSpos | GICP_LIN_REUSE_CORR | GICP_LIN_ERROR_ONLY, corr_a, nullptr)))
                        break;
                }
                const double en = spec ? h[29] : h[27];
                double den = 0.0;
                for (int a = 0; a < 6; ++a) den += delta[a] * (lambda * delta[a] - b[a]);
                const double rho = (e - en) / den;
                if (rho > 0) {
                    std::memcpy(T, Tn, sizeof(T));
                    std::memcpy(piv, pn, sizeof(piv));
                    if (!spec) {  // linearise at the accepted pose now
                        if ((rc = lin(T, piv, corr_b, nullptr))) break;
                    }
                    std::memcpy(lin29, h, sizeof(lin29));
                    std::swap(corr_a, corr_b);
                    std::swap(cache_a, cache_b);
                    const double f = 1.0 - std::pow(2.0 * rho - 1.0, 3);
                    lambda *= (f > 1.0 / 3.0) ? f : 1.0 / 3.0;
                    nu = 2.0;
                    err = en;
                    accepted = true;
                    break;
                }
                lambda *= nu;
                nu *= 2.0;
            }
            if (rc) break;
            if (!accepted) {  // no step decreases the cost: a (numerical) minimum
                converged = 1;
                break;
            }
            done_now = true;  // lin29 already holds the linearisation at the new T
        }
        const double mw = std::fmax(std::fabs(delta[0]), std::fmax(std::fabs(delta[1]), std::fabs(delta[2])));
        const double mv = std::fmax(std::fabs(delta[3]), std::fmax(std::fabs(delta[4]), std::fabs(delta[5])));
        if (debug)
            fprintf(stderr, "[gicp align] it=%d e=%.6f n=%lld lambda=%.3e |dw|=%.3e |dv|=%.3e\n", it, err,
                    (long long)inl, lambda, mw, mv);
        if (debug && cache_a && ns > 0) {  // certificate statistics of the current correspondences
            std::vector<float4> cur((size_t)ns);
            cudaMemcpyAsync(cur.data(), cache_a, ns * sizeof(float4), cudaMemcpyDeviceToHost, s);
            cudaStreamSynchronize(s);
            int64_t valid = 0, kept = 0;
            std::vector<float> rh;
            for (int64_t i = 0; i < ns; ++i) {
                if (cur[i].w > 0.0f) {
                    ++valid;
                    rh.push_back(cur[i].w);
                    if (!dbg_prev.empty() && std::memcmp(&cur[i], &dbg_prev[i], sizeof(float4)) == 0) ++kept;
                }
            }
            std::sort(rh.begin(), rh.end());
            fprintf(stderr, "[gicp align]   certificates valid=%lld carried=%lld rho p10=%.2e p50=%.2e\n",
                    (long long)valid, (long long)kept, rh.empty() ? 0.0 : rh[rh.size() / 10],
                    rh.empty() ? 0.0 : rh[rh.size() / 2]);
            dbg_prev.swap(cur);
        }
        if (mw < prm->rot_eps && mv < prm->trans_eps) {
            converged = 1;
            break;
        }
        if (!done_now) {  // Gauss-Newton: linearise at the new T
            piv[0] = T[3];
            piv[1] = T[7];
            piv[2] = T[11];
            if ((rc = lin(T, piv, corr_a, nullptr)) == GICP_OK) std::memcpy(lin29, h, sizeof(lin29));
        }
    }
    if (kt.used) {
        cudaStreamSynchronize(s);
        kernel_timing_collect(kt);
    }
    cudaFreeAsync(scratch, s);
    std::memcpy(res->T, T, sizeof(T));
    res->iterations = it > prm->max_iter ? prm->max_iter : it;
    res->converged = converged;
    res->error = err;
    res->inliers = inl;
    return rc;
}

// ---- batched registration -----------------------------
// B registrations of concatenated sources against one target in one launch per
// evaluation. Every registration is partitioned into 256-point blocks exactly as
// a single launch over its own points and reduced in the same order, so each
// result is bitwise the single-registration result (tests/test_gpu_parity.py).
namespace gicp {
namespace {

struct BatchScratch {
    char* base = nullptr;
    int4* btab = nullptr;
    int4* ctab = nullptr;   // a round's compacted block table (the active entries' blocks)
    int2* clist = nullptr;  // per active entry: {its first block in btab, its compact start}
    std::vector<int> eblk;  // host: first block of every entry in btab
    int64_t* offs = nullptr;
    Pose* poses = nullptr;
    LinScratch ls;
    int64_t nb = 0;
};

// device scratch: block table, offsets, poses, per-registration counters (+1 for
// the launch), block partials; `extra` bytes appended (16-B aligned) for the caller
int batch_scratch(const int64_t* offsets, int B, size_t extra, cudaStream_t s, BatchScratch& bs, char** extra_p,
                  int nposes = -1) {
    if (nposes < B) nposes = B;
    std::vector<int4> tab;
    for (int b = 0; b < B; ++b) {
        const int64_t n = offsets[b + 1] - offsets[b];
        const int nbk = (int)((n + kLinPPB - 1) / kLinPPB);
        for (int k = 0; k < nbk; ++k) tab.push_back(make_int4(b, k, nbk, (int)tab.size()));
    }
    bs.nb = (int64_t)tab.size();
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    bs.eblk.assign(B + 1, 0);
    for (int b = 0, acc = 0; b <= B; ++b) {
        bs.eblk[b] = acc;
        if (b < B) acc += (int)((offsets[b + 1] - offsets[b] + kLinPPB - 1) / kLinPPB);
    }
    const size_t o_tab = 0, o_offs = al(o_tab + tab.size() * sizeof(int4)), o_pose = al(o_offs + (B + 1) * 8),
                 o_done = al(o_pose + (size_t)nposes * sizeof(Pose)), o_part = al(o_done + (B + 1) * sizeof(unsigned)),
                 o_ctab = al(o_part + linearize_partials_bytes(std::max<int64_t>(bs.nb, 1))),
                 o_clist = al(o_ctab + std::max<size_t>(tab.size(), 1) * sizeof(int4)),
                 o_extra = al(o_clist + (size_t)(B + 1) * sizeof(int2));
    if (cudaMallocAsync((void**)&bs.base, o_extra + extra, s) != cudaSuccess) {
        cudaGetLastError();
        return set_error(GICP_ENOMEM, "batched linearize: scratch allocation failed");
    }
    bs.btab = (int4*)(bs.base + o_tab);
    bs.ctab = (int4*)(bs.base + o_ctab);
    bs.clist = (int2*)(bs.base + o_clist);
    bs.offs = (int64_t*)(bs.base + o_offs);
    bs.poses = (Pose*)(bs.base + o_pose);
    bs.ls.done = (unsigned*)(bs.base + o_done);
    bs.ls.partials = (double*)(bs.base + o_part);
    if (extra_p) *extra_p = bs.base + o_extra;
    int rc = GICP_OK;
    if (!tab.empty())
        rc = check_cuda(cudaMemcpyAsync(bs.btab, tab.data(), tab.size() * sizeof(int4), cudaMemcpyHostToDevice, s),
                        "H2D");
    if (!rc) rc = check_cuda(cudaMemcpyAsync(bs.offs, offsets, (B + 1) * 8, cudaMemcpyHostToDevice, s), "H2D");
    if (!rc) rc = check_cuda(cudaMemsetAsync(bs.ls.done, 0, (B + 1) * sizeof(unsigned), s), "memset");
    // (pageable H2D copies return once the source is staged: the vector may go)
    if (rc) {
        cudaFreeAsync(bs.base, s);
        bs.base = nullptr;
    }
    return rc;
}

int check_offsets(const int64_t* offsets, int B, const char* fn) {
    if (!offsets || B < 1) return set_error(GICP_EINVAL, std::string(fn) + ": offsets / B");
    if (offsets[0] != 0) return set_error(GICP_EINVAL, std::string(fn) + ": offsets[0] must be 0");
    for (int b = 0; b < B; ++b)
        if (offsets[b + 1] < offsets[b]) return set_error(GICP_EINVAL, std::string(fn) + ": offsets not ascending");
    if (offsets[B] >= (1ll << 31) - 1) return set_error(GICP_EINVAL, std::string(fn) + ": too many points");
    return GICP_OK;
}

// host-mapped block of a batched align: B result rows of 32 doubles, the flag,
// and the pinned staging copy of the poses
struct MappedBatch {
    char* h = nullptr;
    char* d = nullptr;
    size_t cap = 0;
};
MappedBatch* mapped_batch(size_t bytes) {
    static thread_local MappedBatch m;
    if (m.cap < bytes) {
        if (m.h) cudaFreeHost(m.h);
        m = MappedBatch{};
        void* p = nullptr;
        if (cudaHostAlloc(&p, bytes, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        void* dp = nullptr;
        if (cudaHostGetDevicePointer(&dp, p, 0) != cudaSuccess) {
            cudaGetLastError();
            cudaFreeHost(p);
            return nullptr;
        }
        std::memset(p, 0, bytes);
        m.h = (char*)p;
        m.d = (char*)dp;
        m.cap = bytes;
    }
    return &m;
}

}  // namespace
}  // namespace gicp

GICP_API int gicp_linearize_batched(const float* src, const float* src_cov, const int64_t* offsets, int B,
                                    gicp_index tgt, const float* tgt_cov, const double* T, const double* pivots,
                                    float max_corr_dist, int flags, double* out29, int32_t* corr, void* stream) {
    int rc;
    if ((rc = check_offsets(offsets, B, "gicp_linearize_batched"))) return rc;
    const int64_t ns = offsets[B];
    if (!tgt || !tgt_cov || !T || !out29) return set_error(GICP_EINVAL, "gicp_linearize_batched: null pointer");
    if (ns > 0 && (!src || !src_cov)) return set_error(GICP_EINVAL, "gicp_linearize_batched: null source");
    if (!(max_corr_dist > 0.0f) || !std::isfinite(max_corr_dist))
        return set_error(GICP_EINVAL, "gicp_linearize_batched: max_corr_dist must be finite and > 0");
    if ((flags & GICP_LIN_REUSE_CORR) && !corr && ns > 0)
        return set_error(GICP_EINVAL, "gicp_linearize_batched: REUSE_CORR needs corr");
    if (flags & ~(GICP_LIN_REUSE_CORR | GICP_LIN_ERROR_ONLY))
        return set_error(GICP_EINVAL, "gicp_linearize_batched: flags");
    for (int b = 0; b < B; ++b) {
        if (!finite_T(T + 16 * b)) return set_error(GICP_EINVAL, "gicp_linearize_batched: non-finite T");
        if (pivots && !(std::isfinite(pivots[3 * b]) && std::isfinite(pivots[3 * b + 1]) &&
                        std::isfinite(pivots[3 * b + 2])))
            return set_error(GICP_EINVAL, "gicp_linearize_batched: non-finite pivot");
    }
    init_pool_once();
    cudaStream_t s = (cudaStream_t)stream;
    if ((rc = check_cuda(cudaMemsetAsync(out29, 0, (size_t)B * 29 * sizeof(double), s), "memset"))) return rc;
    if (ns == 0) return GICP_OK;
    BatchScratch bs;
    if ((rc = batch_scratch(offsets, B, 0, s, bs, nullptr))) return rc;
    std::vector<Pose> poses(B);
    int n_active = 0;
    for (int b = 0; b < B; ++b) {
        poses[b] = make_pose(T + 16 * b, pivots ? pivots + 3 * b : nullptr);
        poses[b].active = offsets[b + 1] > offsets[b];
        n_active += poses[b].active;
    }
    rc = check_cuda(cudaMemcpyAsync(bs.poses, poses.data(), B * sizeof(Pose), cudaMemcpyHostToDevice, s), "H2D");
    if (!rc) {
        BatchView bv;
        bv.btab = bs.btab;
        bv.offs = bs.offs;
        bv.poses = bs.poses;
        bv.n_scans = B;
        bv.n_active = n_active;
        bv.out_stride = 29;
        // one correspondence buffer: current = other = corr (cur = 0, both pointers equal)
        rc = launch_linearize_core(src, src_cov, ns, tgt, tgt_cov, poses[0], max_corr_dist, flags, out29, corr, s,
                                   bs.ls, corr, bv, bs.nb);
    }
    cudaFreeAsync(bs.base, s);
    return rc;
}

// Lockstep LM over B registrations: the per-registration logic is gicp_align's,
// step for step; each evaluation round is ONE batched launch over the
// registrations that need it (the others' blocks exit at once).
// Generalised for sharding: the launch covers E entries (point ranges), entry e
// belonging to registration entry_reg[e]; after every round the entry rows are
// turned into registration rows by `reduce` (a cross-rank combine) or, without
// one, summed in entry order.
// device-side sharding (gicp_align_batched_sharded): entry e is global chunk row
// gid[e] = b * nc + c; rows go through the device chunk table and `ar` (shard.cu)
struct DevShard {
    const int* gid;
    int nc;
    double* table;
    gicp_allreduce_fn ar;
    void* user;
};

static int align_batched_impl(const float* src, const float* src_cov, const int64_t* offsets, int E,
                              const int* entry_reg, int B, gicp_index tgt, const float* tgt_cov, const double* T0,
                              const gicp_align_params* prm, gicp_align_result* res, gicp_reduce_fn reduce,
                              void* user, void* stream, const DevShard* ds = nullptr) {
    int rc;
    std::vector<int> dreg;
    if (ds) {  // the registration of each entry from its global chunk row
        if (ds->nc < 1 || !ds->table || (E > 0 && !ds->gid))
            return set_error(GICP_EINVAL, "gicp_align_batched_sharded: num_chunks / table / entry_chunk");
        dreg.resize(E);
        for (int e = 0; e < E; ++e) {
            if (ds->gid[e] < 0 || ds->gid[e] >= B * ds->nc)
                return set_error(GICP_EINVAL, "gicp_align_batched_sharded: entry_chunk out of range");
            dreg[e] = ds->gid[e] / ds->nc;
        }
        entry_reg = dreg.data();
    }
    if (E == 0 && (reduce || ds)) {  // a process without entries still takes part in the rounds
        if (!offsets || offsets[0] != 0) return set_error(GICP_EINVAL, "gicp_align_batched: offsets");
    } else if ((rc = check_offsets(offsets, E, "gicp_align_batched"))) {
        return rc;
    }
    if (B < 1) return set_error(GICP_EINVAL, "gicp_align_batched: B < 1");
    if (!entry_reg && E != B && E != 0)
        return set_error(GICP_EINVAL, "gicp_align_batched: entry_reg needed when E != B");
    for (int e = 0; entry_reg && e < E; ++e)
        if (entry_reg[e] < 0 || entry_reg[e] >= B) return set_error(GICP_EINVAL, "gicp_align_batched: entry_reg");
    auto reg = [&](int e) { return entry_reg ? entry_reg[e] : e; };
    const int64_t ns = offsets[E];
    if (!tgt || !tgt_cov || !T0 || !prm || !res || (ns > 0 && (!src || !src_cov)))
        return set_error(GICP_EINVAL, "gicp_align_batched: null pointer");
    if (prm->max_iter < 1) return set_error(GICP_EINVAL, "gicp_align_batched: max_iter < 1");
    for (int b = 0; b < B; ++b)
        if (!finite_T(T0 + 16 * b)) return set_error(GICP_EINVAL, "gicp_align_batched: non-finite T0");
    init_pool_once();
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t nsa = ns > 0 ? ns : 1;
    // device: batch scratch + two correspondence buffers + the sorted source copy
    BatchScratch bs;
    char* ex = nullptr;
    // + the correspondence certificates paired with the two buffers (R27)
    const bool certs = GICP_ALIGN_CACHE && getenv("GICP_ALIGN_NOCACHE") == nullptr;
    const size_t dev_extra = (ds ? (size_t)std::max(E, 1) * (32 * sizeof(double) + sizeof(int)) : 0) +
                             (size_t)std::max(E, 1) * sizeof(int) + 768;
    if ((rc = batch_scratch(offsets, E,
                            2 * nsa * sizeof(int32_t) + nsa * 9 * sizeof(float) + 64 +
                                (certs ? 4 * nsa * sizeof(float4) + 64 : 0) + dev_extra,
                            s, bs, &ex, B)))
        return rc;
    double* Ed = nullptr;  // device entry rows [E][32] (device sharding)
    int* gid_d = nullptr;
    // entry -> registration (the poses go up per registration, not per entry)
    int* ereg_d = (int*)(((uintptr_t)ex + 2 * nsa * sizeof(int32_t) + nsa * 9 * sizeof(float) + 64 +
                          (certs ? 4 * nsa * sizeof(float4) + 64 : 0) + 255) & ~(uintptr_t)255);
    if (ds) {
        Ed = (double*)(((uintptr_t)(ereg_d + std::max(E, 1)) + 255) & ~(uintptr_t)255);
        gid_d = (int*)(Ed + 32 * (size_t)std::max(E, 1));
        if (E > 0 &&
            (rc = check_cuda(cudaMemcpyAsync(gid_d, ds->gid, E * sizeof(int), cudaMemcpyHostToDevice, s), "H2D"))) {
            cudaFreeAsync(bs.base, s);
            return rc;
        }
    }
    if (E > 0) {
        std::vector<int> er(E);
        for (int e = 0; e < E; ++e) er[e] = entry_reg ? entry_reg[e] : e;
        if ((rc = check_cuda(cudaMemcpyAsync(ereg_d, er.data(), E * sizeof(int), cudaMemcpyHostToDevice, s), "H2D"))) {
            cudaFreeAsync(bs.base, s);
            return rc;
        }
    }
    int32_t* corrA = (int32_t*)ex;
    int32_t* corrB = corrA + nsa;
    float* src_p = (float*)(((uintptr_t)(corrB + nsa) + 15) & ~(uintptr_t)15);
    float* cov_p = (float*)(((uintptr_t)(src_p + 3 * nsa) + 15) & ~(uintptr_t)15);  // float2 loads
    if (certs) {  // cache_new pairs with corrA, cache_old with corrB; the kernel maps them per `cur`
        bs.ls.cache_new = (float4*)(((uintptr_t)(cov_p + 6 * nsa) + 15) & ~(uintptr_t)15);
        bs.ls.cache_old = bs.ls.cache_new + nsa;
        if (split_eval(nsa)) {  // the split evaluation's search queue and counter
            bs.ls.queue = bs.ls.cache_new + 2 * nsa;
            bs.ls.queue2 = bs.ls.queue + nsa;
            bs.ls.qcount = (unsigned*)(bs.ls.queue2 + nsa);
        }
    }
    if (ns > 0 && (rc = sort_source(src, src_cov, ns, tgt->lv[0].cell, src_p, cov_p, s, bs.offs, E))) {
        cudaFreeAsync(bs.base, s);
        return rc;
    }
    // host-mapped: entry rows [E][32] (device sharding: registration rows [B][32]) |
    // flag | pinned pose staging [E]
    const size_t rows = (size_t)(ds ? std::max(E, B) : E) * 32 * sizeof(double);
    MappedBatch* mb = mapped_batch(rows + 256 + (size_t)std::max(E, B) * sizeof(Pose) + 3 * (size_t)(E + 1) * sizeof(int2));
    if (!mb) {
        cudaFreeAsync(bs.base, s);
        return set_error(GICP_ENOMEM, "gicp_align_batched: host-mapped buffer");
    }
    double* He = (double*)mb->h;
    double* Hd = (double*)mb->d;
    volatile unsigned* hflag = (volatile unsigned*)(mb->h + rows);
    Pose* pst = (Pose*)(mb->h + rows + 256);
    static thread_local unsigned seq = 0;
    MappedOut mo;  // wait_mapped view of the flag
    mo.flag = hflag;
    bs.ls.flag = (volatile unsigned*)(mb->d + rows);
    std::vector<double> Hr((size_t)B * 32, 0.0);  // registration rows of the last round
    const double* H = Hr.data();

    // Per-registration state machine (each registration takes exactly the evaluation
    // sequence of gicp_align on it alone; a round evaluates every unfinished
    // registration once, whatever its next evaluation is, so slow registrations no
    // longer hold the others in lockstep): FULL = linearise at T (initial, or after a
    // trial accepted), DUAL = the speculative first trial of an iteration (the full
    // linearisation at Tn plus e' with the current correspondences), TRIAL = e' alone
    // at Tn (a later trial after a rejection).
    enum { M_DONE = 0, M_FULL = 1, M_DUAL = 2, M_TRIAL = 3 };
    struct St {
        double T[16], piv[3], lin29[29], Tn[16], pn[3], delta[6], Hm[36], b[6];
        double lambda = -1.0, nu = 2.0, err = 0.0, e = 0.0;
        double disp = INFINITY;  // the last step's point motion (kLinCoarse)
        int it = 0, converged = 0, cur = 0, rc = GICP_OK, inner = 0, mode = M_FULL;
        int relin = 0;           // a FULL after an accepted trial (LM: test convergence after it)
        int64_t inl = 0;
    };
    std::vector<St> st(B);
    for (int b = 0; b < B; ++b) {
        std::memcpy(st[b].T, T0 + 16 * b, sizeof(st[b].T));
        st[b].piv[0] = st[b].T[3];
        st[b].piv[1] = st[b].T[7];
        st[b].piv[2] = st[b].T[11];
        if (!reduce && !ds && !entry_reg && offsets[b + 1] == offsets[b]) {  // no points: no correspondences
            st[b].mode = M_DONE;
            st[b].rc = GICP_EDEGENERATE;
        }
    }
    // the level-1 cube stage after the first evaluation: the split evaluation (>= 1M
    // points, linearize.cu) settles far points in its cooperative full pass, so there
    // only the first evaluation (pose error unknown) takes it (C4 dual launch 0.89 ->
    // 0.86 ms against the single-align threshold); GICP_LIN_COARSE_FIRST=0 not even that
    int64_t split_min = 1 << 20;
    if (const char* e = getenv("GICP_LIN_SPLIT_MIN")) split_min = atoll(e);
    const bool split_path = ns >= split_min;
    const double coarse_thr = split_path ? 1e300 : coarse_threshold(tgt);
    static const bool coarse_first = !(getenv("GICP_LIN_COARSE_FIRST") && atoi(getenv("GICP_LIN_COARSE_FIRST")) == 0);
    // GICP_DEBUG_ALIGN_HOST: rounds, their device-wait time and the host time between them
    const bool host_trace = getenv("GICP_DEBUG_ALIGN_HOST") != nullptr;
    using clk = std::chrono::steady_clock;
    double t_wait = 0.0, t_total = 0.0;
    int n_rounds = 0, n_launch = 0;
    const auto t_begin = clk::now();
    std::vector<char> eact(std::max(E, 1));
    // one round: every unfinished registration evaluated once; one launch per kind
    // present (a compacted block table of that kind's entries), then the rows (the
    // device chunk table + allreduce + combine when sharded). Every rank calls the
    // collective on every round (collectives stay matched) even when it launches nothing.
    auto round = [&]() -> int {
        ++n_rounds;
        int n_any = 0;
        for (int b = 0; b < B; ++b) {
            const St& q = st[b];
            pst[b].active = q.mode != M_DONE;
            if (q.mode == M_DONE) continue;
            const bool trial = q.mode == M_DUAL || q.mode == M_TRIAL;
            pst[b] = make_pose(trial ? q.Tn : q.T, trial ? q.pn : q.piv);
            pst[b].active = 1;
            pst[b].cur = q.cur;
            pst[b].coarse = q.disp > coarse_thr && (coarse_first || !split_path);  // per registration (§4.3)
        }
        for (int e = 0; e < E; ++e) n_any += pst[reg(e)].active && offsets[e + 1] > offsets[e];
        int r = GICP_OK;
        unsigned last_seq = 0;
        if (n_any > 0) {
            r = check_cuda(cudaMemcpyAsync(bs.poses, pst, B * sizeof(Pose), cudaMemcpyHostToDevice, s), "H2D");
            if (r) return r;
            for (int kind = M_FULL; kind <= M_TRIAL; ++kind) {
                int n_active = 0;
                for (int e = 0; e < E; ++e) {
                    eact[e] = offsets[e + 1] > offsets[e] && st[reg(e)].mode == kind;  // an empty entry has no block
                    n_active += eact[e];
                }
                if (!n_active) continue;
                const int flags = kind == M_FULL ? kLinCorrSpos
                                  : kind == M_DUAL ? (kLinCorrSpos | kLinDual)
                                                   : (kLinCorrSpos | GICP_LIN_REUSE_CORR | GICP_LIN_ERROR_ONLY);
                BatchView bv;
                bv.btab = bs.btab;
                bv.offs = bs.offs;
                bv.poses = bs.poses;
                bv.ereg = ereg_d;
                bv.n_scans = E;
                bv.n_active = n_active;
                bv.out_stride = 32;
                int64_t nbl = bs.nb;
                // this kind's entries as a {first block, compact start} list (pinned
                // staging, one region per kind): the deferred reduction's entries
                // and, when only part of the entries is active, the compacted block
                // table (expanded on the device) that launches only their blocks
                int2* cl = (int2*)(mb->h + rows + 256 + (size_t)std::max(E, B) * sizeof(Pose)) +
                           (size_t)(kind - 1) * (E + 1);
                int nce = 0, acc = 0;
                for (int e = 0; e < E; ++e)
                    if (eact[e]) {
                        cl[nce++] = make_int2(bs.eblk[e], acc);
                        acc += bs.eblk[e + 1] - bs.eblk[e];
                    }
                cl[nce] = make_int2(0, acc);
                r = check_cuda(cudaMemcpyAsync(bs.clist, cl, (nce + 1) * sizeof(int2), cudaMemcpyHostToDevice, s),
                               "H2D");
                if (r) return r;
                if (n_active < E) {
                    r = launch_compact_btab(bs.btab, bs.clist, nce, acc, bs.ctab, s);
                    if (r) return r;
                    bv.btab = bs.ctab;
                    nbl = acc;
                }
                if (deferred_reduce()) {
                    bv.elist = bs.clist;
                    bv.n_e = nce;
                    bv.btab_full = bs.btab;
                }
                bs.ls.seq = ++seq;
                last_seq = bs.ls.seq;
                LinScratch lsr = bs.ls;
                if (ds) lsr.flag = nullptr;  // the combine kernel signals
                KernelTiming& kt = kernel_timing();
                const bool timed = kt.on && kt.used < KernelTiming::kCap;
                if (timed) cudaEventRecord(kt.e[2 * kt.used], s);
                ++n_launch;
                r = launch_linearize_core(src_p, cov_p, ns, tgt, tgt_cov, pst[0], prm->max_corr_dist, flags,
                                          ds ? Ed : Hd, corrA, s, lsr, corrB, bv, nbl);
                if (timed) {
                    cudaEventRecord(kt.e[2 * kt.used + 1], s);
                    int64_t ap = 0;
                    for (int e = 0; e < E; ++e)
                        if (eact[e]) ap += offsets[e + 1] - offsets[e];
                    kt.lpts[kt.used] = ap;
                    kt.kind[kt.used++] = kind == M_DUAL ? 0 : (kind == M_TRIAL ? 2 : 1);
                }
                if (r) return r;
            }
            if (!ds) {
                const auto w0 = clk::now();
                r = wait_mapped(&mo, last_seq, s);
                t_wait += std::chrono::duration<double, std::milli>(clk::now() - w0).count();
                if (r) return r;
            }
        }
        for (int e = 0; e < E; ++e) eact[e] = pst[reg(e)].active && offsets[e + 1] > offsets[e];
        if (ds) {
            // device chunk table: zero, this rank's rows, allreduce, chunk-ordered combine
            const size_t tb = (size_t)B * ds->nc * 32 * sizeof(double);
            r = check_cuda(cudaMemsetAsync(ds->table, 0, tb, s), "memset");
            if (!r && n_any > 0) r = launch_scatter_rows(Ed, E, gid_d, ereg_d, bs.poses, bs.offs, ds->table, s);
            if (!r && ds->ar && ds->ar(ds->table, (int64_t)B * ds->nc * 32, ds->user, stream) != 0)
                r = set_error(GICP_ECUDA, "gicp_align_batched_sharded: the allreduce callback failed");
            if (r) return r;
            bs.ls.seq = ++seq;
            r = launch_combine_chunks(ds->table, B, ds->nc, 32, Hd, bs.ls.flag, bs.ls.seq, s);
            const auto w0 = clk::now();
            if (!r) r = wait_mapped(&mo, bs.ls.seq, s);
            t_wait += std::chrono::duration<double, std::milli>(clk::now() - w0).count();
            if (r) return r;
            std::memcpy(Hr.data(), He, (size_t)B * 32 * sizeof(double));
            return GICP_OK;
        }
        for (int e = 0; e < E; ++e)  // rows of entries not launched this round are zero
            if (!eact[e]) std::memset(He + 32 * e, 0, 32 * sizeof(double));
        if (reduce) {
            if (reduce(He, E, Hr.data(), B, user) != 0)
                return set_error(GICP_ECUDA, "gicp_align_batched: the reduce callback failed");
        } else {
            std::fill(Hr.begin(), Hr.end(), 0.0);
            for (int e = 0; e < E; ++e)
                for (int c = 0; c < 32; ++c) Hr[32 * reg(e) + c] += He[32 * e + c];
        }
        return GICP_OK;
    };
    auto converged_step = [&](const St& q) {
        const double mw = std::fmax(std::fabs(q.delta[0]), std::fmax(std::fabs(q.delta[1]), std::fabs(q.delta[2])));
        const double mv = std::fmax(std::fabs(q.delta[3]), std::fmax(std::fabs(q.delta[4]), std::fabs(q.delta[5])));
        return mw < prm->rot_eps && mv < prm->trans_eps;
    };
    // the next trial of an LM iteration (DUAL for the first, TRIAL after a rejection);
    // ten solves / trials without an accepted step: a (numerical) minimum
    auto try_trial = [&](St& q) {
        while (q.inner < 10) {
            double Hl[36], nb[6];
            std::memcpy(Hl, q.Hm, sizeof(Hl));
            for (int a = 0; a < 6; ++a) {
                Hl[7 * a] += q.lambda;
                nb[a] = -q.b[a];
            }
            if (!ldlt6(Hl, nb, q.delta)) {
                q.lambda *= q.nu;
                q.nu *= 2.0;
                ++q.inner;
                continue;
            }
            double Em[16];
            pivoted_exp(q.delta, q.piv, Em);
            q.disp = step_displacement(q.delta);
            mul44(Em, q.T, q.Tn);
            q.pn[0] = q.Tn[3];
            q.pn[1] = q.Tn[7];
            q.pn[2] = q.Tn[11];
            q.mode = q.inner == 0 ? M_DUAL : M_TRIAL;
            return;
        }
        q.converged = 1;
        q.mode = M_DONE;
    };
    // a new iteration from the linearisation at T (lin29)
    auto start_iteration = [&](St& q) {
        if (++q.it > prm->max_iter) {
            q.it = prm->max_iter;
            q.mode = M_DONE;
            return;
        }
        q.inl = (int64_t)q.lin29[28];
        if (q.inl < 6) {
            q.rc = GICP_EDEGENERATE;
            q.mode = M_DONE;
            return;
        }
        for (int a = 0, o = 0; a < 6; ++a)
            for (int c = a; c < 6; ++c, ++o) q.Hm[6 * a + c] = q.Hm[6 * c + a] = q.lin29[o];
        for (int a = 0; a < 6; ++a) q.b[a] = q.lin29[21 + a];
        q.e = q.lin29[27];
        q.err = q.e;
        for (int a = 0; a < 6; ++a) q.delta[a] = 0.0;
        if (!prm->lm) {  // Gauss-Newton: the step, its convergence test, then re-linearise
            double nb[6];
            for (int a = 0; a < 6; ++a) nb[a] = -q.b[a];
            if (!ldlt6(q.Hm, nb, q.delta)) {
                q.rc = GICP_EDEGENERATE;
                q.mode = M_DONE;
                return;
            }
            double Em[16];
            pivoted_exp(q.delta, q.piv, Em);
            q.disp = step_displacement(q.delta);
            mul44(Em, q.T, q.T);
            if (converged_step(q)) {
                q.converged = 1;
                q.mode = M_DONE;
                return;
            }
            q.piv[0] = q.T[3];
            q.piv[1] = q.T[7];
            q.piv[2] = q.T[11];
            q.relin = 0;
            q.mode = M_FULL;
            return;
        }
        if (q.lambda < 0) {
            double mx = 0.0;
            for (int a = 0; a < 6; ++a) mx = std::fmax(mx, q.Hm[7 * a]);
            q.lambda = 1e-9 * mx;
        }
        q.inner = 0;
        try_trial(q);
    };
    auto accept = [&](St& q, double rho, double en) {
        std::memcpy(q.T, q.Tn, sizeof(q.T));
        std::memcpy(q.piv, q.pn, sizeof(q.piv));
        const double f = 1.0 - std::pow(2.0 * rho - 1.0, 3);
        q.lambda *= (f > 1.0 / 3.0) ? f : 1.0 / 3.0;
        q.nu = 2.0;
        q.err = en;
    };
    auto reject = [&](St& q) {
        q.lambda *= q.nu;
        q.nu *= 2.0;
        ++q.inner;
        try_trial(q);
    };
    const bool dbg_rows = getenv("GICP_DEBUG_ALIGN") != nullptr;
    while (!rc) {
        bool any = false;
        for (int b = 0; b < B; ++b) any |= st[b].mode != M_DONE;
        if (!any) break;
        if ((rc = round())) break;
        if (dbg_rows)
            for (int b = 0; b < B; ++b)
                if (st[b].mode != M_DONE)
                    fprintf(stderr, "[gicp align_batched] round %d reg %d mode %d it %d: H00 %.9g b0 %.9g e %.9g n %.0f "
                            "e' %.9g\n", n_rounds, b, st[b].mode, st[b].it, Hr[32 * b], Hr[32 * b + 21], Hr[32 * b + 27],
                            Hr[32 * b + 28], Hr[32 * b + 29]);
        for (int b = 0; b < B; ++b) {
            St& q = st[b];
            const double* h = Hr.data() + 32 * b;
            switch (q.mode) {
                case M_FULL: {  // a linearisation at T: the other correspondence buffer becomes current
                    std::memcpy(q.lin29, h, sizeof(q.lin29));
                    q.cur ^= 1;
                    if (q.relin && prm->lm && converged_step(q)) {
                        q.converged = 1;
                        q.mode = M_DONE;
                        break;
                    }
                    q.relin = 0;
                    start_iteration(q);
                    break;
                }
                case M_DUAL: {
                    const double en = h[29];
                    double den = 0.0;
                    for (int a = 0; a < 6; ++a) den += q.delta[a] * (q.lambda * q.delta[a] - q.b[a]);
                    const double rho = (q.e - en) / den;
                    if (rho > 0) {  // the speculative full linearisation at Tn is kept
                        accept(q, rho, en);
                        std::memcpy(q.lin29, h, sizeof(q.lin29));
                        q.cur ^= 1;
                        if (converged_step(q)) {
                            q.converged = 1;
                            q.mode = M_DONE;
                        } else {
                            start_iteration(q);
                        }
                    } else {
                        reject(q);
                    }
                    break;
                }
                case M_TRIAL: {
                    const double en = h[27];
                    double den = 0.0;
                    for (int a = 0; a < 6; ++a) den += q.delta[a] * (q.lambda * q.delta[a] - q.b[a]);
                    const double rho = (q.e - en) / den;
                    if (rho > 0) {  // accepted: linearise at the new pose, then test convergence
                        accept(q, rho, en);
                        q.relin = 1;
                        q.mode = M_FULL;
                    } else {
                        reject(q);
                    }
                    break;
                }
                default:
                    break;
            }
        }
    }
    t_total = std::chrono::duration<double, std::milli>(clk::now() - t_begin).count();
    if (host_trace)
        fprintf(stderr, "[gicp align_batched host] B=%d E=%d rounds=%d launches=%d total %.2f ms, waiting on the device "
                "%.2f ms\n", B, E, n_rounds, n_launch, t_total, t_wait);
    cudaFreeAsync(bs.base, s);
    {
        KernelTiming& kt = kernel_timing();
        if (kt.used) {
            cudaStreamSynchronize(s);
            kernel_timing_collect(kt);
        }
    }
    int any_degenerate = 0;
    for (int b = 0; b < B; ++b) {
        std::memcpy(res[b].T, st[b].T, sizeof(res[b].T));
        res[b].iterations = st[b].it;
        res[b].converged = st[b].converged;
        res[b].error = st[b].err;
        res[b].inliers = st[b].inl;
        any_degenerate |= st[b].rc == GICP_EDEGENERATE;
    }
    if (rc) return rc;
    return any_degenerate ? set_error(GICP_EDEGENERATE, "gicp_align_batched: a registration has < 6 correspondences")
                          : GICP_OK;
}

GICP_API int gicp_align_batched(const float* src, const float* src_cov, const int64_t* offsets, int B,
                                gicp_index tgt, const float* tgt_cov, const double* T0,
                                const gicp_align_params* prm, gicp_align_result* res, void* stream) {
    return align_batched_impl(src, src_cov, offsets, B, nullptr, B, tgt, tgt_cov, T0, prm, res, nullptr, nullptr,
                              stream);
}

GICP_API int gicp_align_batched_sharded(const float* src, const float* src_cov, const int64_t* offsets, int E,
                                        const int* entry_chunk, int num_chunks, int B, gicp_index tgt,
                                        const float* tgt_cov, const double* T0, const gicp_align_params* prm,
                                        gicp_align_result* res, double* table, gicp_allreduce_fn allreduce,
                                        void* user, void* stream) {
    const DevShard ds{entry_chunk, num_chunks, table, allreduce, user};
    return align_batched_impl(src, src_cov, offsets, E, nullptr, B, tgt, tgt_cov, T0, prm, res, nullptr, nullptr,
                              stream, &ds);
}

GICP_API int gicp_combine_chunks(const double* table, int B, int num_chunks, int width, double* out, void* stream) {
    if (!table || !out || B < 0 || num_chunks < 1 || width < 1)
        return set_error(GICP_EINVAL, "gicp_combine_chunks: arguments");
    if (B == 0) return GICP_OK;
    init_pool_once();
    return launch_combine_chunks(table, B, num_chunks, width, out, nullptr, 0u, (cudaStream_t)stream);
}

GICP_API int gicp_align_batched_ex(const float* src, const float* src_cov, const int64_t* offsets, int E,
                                   const int* entry_reg, int B, gicp_index tgt, const float* tgt_cov,
                                   const double* T0, const gicp_align_params* prm, gicp_align_result* res,
                                   gicp_reduce_fn reduce, void* user, void* stream) {
    return align_batched_impl(src, src_cov, offsets, E, entry_reg, B, tgt, tgt_cov, T0, prm, res, reduce, user,
                              stream);
}

// ---- voxelized GICP ---------------------------------------

GICP_API int gicp_index_attach_voxels(gicp_index idx, const float* cov, void* stream) {
    if (!idx || !cov) return set_error(GICP_EINVAL, "gicp_index_attach_voxels: null pointer");
    init_pool_once();
    return attach_voxels(idx, cov, (cudaStream_t)stream);
}

GICP_API int gicp_linearize_vgicp(const float* src, const float* src_cov, int64_t ns, gicp_index tgt,
                                  const double T[16], const double* pivot, int mode, int flags, int32_t* base,
                                  double* out29, void* stream) {
    if (!tgt || !T || !out29) return set_error(GICP_EINVAL, "gicp_linearize_vgicp: null pointer");
    if (!tgt->vox_mu) return set_error(GICP_EINVAL, "gicp_linearize_vgicp: call gicp_index_attach_voxels first");
    if (ns < 0 || ns >= (1ll << 31) - 1) return set_error(GICP_EINVAL, "gicp_linearize_vgicp: ns out of range");
    if (ns > 0 && (!src || !src_cov)) return set_error(GICP_EINVAL, "gicp_linearize_vgicp: null source");
    if (mode != 1 && mode != 7 && mode != 27) return set_error(GICP_EINVAL, "gicp_linearize_vgicp: mode 1, 7 or 27");
    if (flags & ~(GICP_LIN_ERROR_ONLY | GICP_LIN_REUSE_CORR)) return set_error(GICP_EINVAL, "gicp_linearize_vgicp: flags");
    if ((flags & GICP_LIN_REUSE_CORR) && !base && ns > 0)
        return set_error(GICP_EINVAL, "gicp_linearize_vgicp: REUSE_CORR needs base");
    if (!finite_T(T)) return set_error(GICP_EINVAL, "gicp_linearize_vgicp: non-finite T");
    init_pool_once();
    return launch_linearize_vgicp(src, src_cov, ns, tgt, T, pivot, mode, flags, base, out29, (cudaStream_t)stream);
}

// LM on the voxelized linearisation with gicp_align's schedule (R13); the trial
// cost keeps the pairs (base voxels) of the linearisation (reading R23).
GICP_API int gicp_align_vgicp(const float* src, const float* src_cov, int64_t ns, gicp_index tgt, int mode,
                              const double T0[16], const gicp_align_params* prm, gicp_align_result* res,
                              void* stream) {
    if (!tgt || !T0 || !prm || !res || (ns > 0 && (!src || !src_cov)))
        return set_error(GICP_EINVAL, "gicp_align_vgicp: null pointer");
    if (!tgt->vox_mu) return set_error(GICP_EINVAL, "gicp_align_vgicp: call gicp_index_attach_voxels first");
    if (mode != 1 && mode != 7 && mode != 27) return set_error(GICP_EINVAL, "gicp_align_vgicp: mode 1, 7 or 27");
    if (prm->max_iter < 1) return set_error(GICP_EINVAL, "gicp_align_vgicp: max_iter < 1");
    if (!finite_T(T0)) return set_error(GICP_EINVAL, "gicp_align_vgicp: non-finite T0");
    init_pool_once();
    cudaStream_t s = (cudaStream_t)stream;
    MappedOut* mo = mapped_out();
    if (!mo) return set_error(GICP_ENOMEM, "gicp_align_vgicp: host-mapped buffer");
    const size_t bytes = 512 + vgicp_scratch_bytes(ns > 0 ? ns : 1) + 3 * sizeof(int) * (ns > 0 ? ns : 1) + 16;
    char* scratch = nullptr;
    if (cudaMallocAsync((void**)&scratch, bytes, s) != cudaSuccess) {
        cudaGetLastError();
        return set_error(GICP_ENOMEM, "gicp_align_vgicp: scratch allocation failed");
    }
    LinScratch ls;
    ls.done = (unsigned*)(scratch + 256);
    ls.partials = (double*)(scratch + 512);
    double* d_out = (double*)scratch;
    int* base = (int*)(((uintptr_t)(scratch + 512 + vgicp_scratch_bytes(ns > 0 ? ns : 1)) + 15) & ~(uintptr_t)15);
    int rc = check_cuda(cudaMemsetAsync(ls.done, 0, sizeof(unsigned), s), "memset");
    double h[29];
    auto lin = [&](const double* T, const double* piv, int flags) -> int {
        int r = launch_linearize_vgicp(src, src_cov, ns, tgt, T, piv, mode, flags, base, d_out, s, &ls);
        if (!r) r = read_small(h, d_out, sizeof(h), s);
        return r;
    };
    double T[16];
    std::memcpy(T, T0, sizeof(T));
    double lambda = -1.0, nu = 2.0, err = 0.0;
    int converged = 0, it = 0;
    int64_t inl = 0;
    for (it = 1; !rc && it <= prm->max_iter; ++it) {
        const double piv[3] = {T[3], T[7], T[11]};
        if ((rc = lin(T, piv, 0))) break;
        inl = (int64_t)h[28];
        if (inl < 6) {
            rc = set_error(GICP_EDEGENERATE, "gicp_align_vgicp: fewer than 6 voxel pairs");
            break;
        }
        double Hm[36], b[6], delta[6] = {0, 0, 0, 0, 0, 0};
        for (int a = 0, o = 0; a < 6; ++a)
            for (int c = a; c < 6; ++c, ++o) Hm[6 * a + c] = Hm[6 * c + a] = h[o];
        for (int a = 0; a < 6; ++a) b[a] = h[21 + a];
        const double e = h[27];
        err = e;
        if (lambda < 0) {
            double mx = 0.0;
            for (int a = 0; a < 6; ++a) mx = std::fmax(mx, Hm[7 * a]);
            lambda = 1e-9 * mx;
        }
        bool accepted = false;
        for (int inner = 0; inner < 10; ++inner) {
            double Hl[36], nb[6];
            std::memcpy(Hl, Hm, sizeof(Hl));
            for (int a = 0; a < 6; ++a) {
                Hl[7 * a] += lambda;
                nb[a] = -b[a];
            }
            if (!ldlt6(Hl, nb, delta)) {
                lambda *= nu;
                nu *= 2.0;
                continue;
            }
            double E[16], Tn[16];
            pivoted_exp(delta, piv, E);
            mul44(E, T, Tn);
            const double pn[3] = {Tn[3], Tn[7], Tn[11]};
            if ((rc = lin(Tn, pn, GICP_LIN_ERROR_ONLY | GICP_LIN_REUSE_CORR))) break;
            const double en = h[27];
            double den = 0.0;
            for (int a = 0; a < 6; ++a) den += delta[a] * (lambda * delta[a] - b[a]);
            const double rho = (e - en) / den;
            if (rho > 0) {
                std::memcpy(T, Tn, sizeof(T));
                const double f = 1.0 - std::pow(2.0 * rho - 1.0, 3);
                lambda *= (f > 1.0 / 3.0) ? f : 1.0 / 3.0;
                nu = 2.0;
                err = en;
                accepted = true;
                break;
            }
            lambda *= nu;
            nu *= 2.0;
        }
        if (rc) break;
        if (!accepted) {
            converged = 1;
            break;
        }
        const double mw = std::fmax(std::fabs(delta[0]), std::fmax(std::fabs(delta[1]), std::fabs(delta[2])));
        const double mv = std::fmax(std::fabs(delta[3]), std::fmax(std::fabs(delta[4]), std::fabs(delta[5])));
        if (mw < prm->rot_eps && mv < prm->trans_eps) {
            converged = 1;
            break;
        }
    }
    cudaFreeAsync(scratch, s);
    std::memcpy(res->T, T, sizeof(T));
    res->iterations = it > prm->max_iter ? prm->max_iter : it;
    res->converged = converged;
    res->error = err;
    res->inliers = inl;
    return rc;
}

// ---- z-vote ground filter -----------------------------------
GICP_API int gicp_ground_filter(const float* xyz, int64_t n, float cell, int min_count, uint8_t* keep, int32_t* count,
                                void* stream) {
    if (n < 0) return set_error(GICP_EINVAL, "gicp_ground_filter: n < 0");
    if (!(cell > 0.0f) || !std::isfinite(cell)) return set_error(GICP_EINVAL, "gicp_ground_filter: cell must be > 0");
    if (n > 0 && (!xyz || !keep)) return set_error(GICP_EINVAL, "gicp_ground_filter: null pointer");
    init_pool_once();
    return launch_ground_filter(xyz, n, cell, min_count, keep, count, (cudaStream_t)stream);
}

// ---- Euclidean cluster extraction ----------------------------
GICP_API int gicp_cluster(const float* xyz, int64_t n, float tol, int min_size, int32_t* label, int64_t* n_clusters,
                          void* stream) {
    if (!n_clusters || n < 0 || (n > 0 && (!xyz || !label))) return set_error(GICP_EINVAL, "gicp_cluster: null / n");
    if (!(tol > 0.0f) || !std::isfinite(tol)) return set_error(GICP_EINVAL, "gicp_cluster: tol must be > 0");
    if (n >= (1ll << 31) - 1) return set_error(GICP_EINVAL, "gicp_cluster: n too large");
    init_pool_once();
    return launch_cluster(xyz, n, tol, min_size, label, n_clusters, (cudaStream_t)stream);
}

// ---- diagnostics ----------------------------------------------------------------
GICP_API int gicp_align_timing(int enable, double* ms /* host [3] or NULL */, int64_t* launches /* host [3] */,
                               int64_t* points /* host [3] */) {
    KernelTiming& t = kernel_timing();
    if (ms)
        for (int k = 0; k < 3; ++k) ms[k] = t.ms[k];
    if (launches)
        for (int k = 0; k < 3; ++k) launches[k] = t.n[k];
    if (points)
        for (int k = 0; k < 3; ++k) points[k] = t.pts[k];
    for (int k = 0; k < 3; ++k) {
        t.ms[k] = 0.0;
        t.n[k] = 0;
        t.pts[k] = 0;
    }
    if (enable && !t.e[0]) {
        for (auto& ev : t.e)
            if (cudaEventCreate(&ev) != cudaSuccess) {
                cudaGetLastError();
                return set_error(GICP_ECUDA, "gicp_align_timing: event creation failed");
            }
    }
    t.on = enable ? 1 : 0;
    return GICP_OK;
}
