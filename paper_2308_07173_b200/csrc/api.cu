// api.cu -- the extern "C" boundary of libgicp_b200 (declared in include/gicp.h):
// argument validation, thread-local errors, and the host LM loop of gicp_align.
#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "gicp_internal.cuh"

#define GICP_API extern "C" __attribute__((visibility("default")))

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
    double z[6];
    for (int i = 0; i < 6; ++i) {
        double s = y[i];
        for (int p = 0; p < i; ++p) s -= L[i][p] * z[p];
        z[i] = s / D[i];
    }
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

}  // namespace
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
    cudaGetLastError();
    delete idx;
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

GICP_API int gicp_align(const float* src, const float* src_cov, int64_t ns, gicp_index tgt, const float* tgt_cov,
                        const double T0[16], const gicp_align_params* prm, gicp_align_result* res, void* stream) {
    if (!tgt || !tgt_cov || !T0 || !prm || !res || (ns > 0 && (!src || !src_cov)))
        return set_error(GICP_EINVAL, "gicp_align: null pointer");
    if (ns < 0) return set_error(GICP_EINVAL, "gicp_align: ns < 0");
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
    const size_t bytes = 512 + lin_bytes + 2 * nsa * sizeof(int32_t) + nsa * 9 * sizeof(float) + 256;
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
    float* cov_p = src_p + 3 * nsa;
    int rc0 = check_cuda(cudaMemsetAsync(ls.done, 0, sizeof(unsigned), s), "memset");
    if (!rc0 && ns > 0) rc0 = sort_source(src, src_cov, ns, tgt->lv[0].cell, src_p, cov_p, s);
    if (rc0) {
        cudaFreeAsync(scratch, s);
        return rc0;
    }
    // one launch + one sync per evaluation: `old` != nullptr also evaluates the
    // trial cost with the previous correspondences (values 29, 30)
    ls.flag = mo->dflag;
    auto go = [&](const double* T, const double* piv, int flags, int32_t* corr, const int32_t* old) -> int {
        ls.seq = ++mo->seq;
        const int rc = launch_linearize(src_p, cov_p, ns, tgt, tgt_cov, T, piv, prm->max_corr_dist, flags, mo->d,
                                        corr, s, &ls, old);
        return rc ? rc : wait_mapped(mo, ls.seq, s);
    };
    auto lin = [&](const double* T, const double* piv, int32_t* corr, const int32_t* old) -> int {
        return go(T, piv, kLinCorrSpos, corr, old);
    };
    const bool debug = getenv("GICP_DEBUG_ALIGN") != nullptr;
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
    cudaFreeAsync(scratch, s);
    std::memcpy(res->T, T, sizeof(T));
    res->iterations = it > prm->max_iter ? prm->max_iter : it;
    res->converged = converged;
    res->error = err;
    res->inliers = inl;
    return rc;
}
