/*
 * oracle.c -- the plain, slow, obviously-correct CPU ORACLE for the GICP hot path.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load or call this library. The product
 * path (paper_2308_07173_b200/) never links, imports or executes it, and this file
 * shares no code, header, table or constant generator with the CUDA sources.
 *
 * What it computes (the "plain definitions" of SURVEY.md §8(c) O1-O4; readings
 * of the paper are listed in DESIGN.md §Readings):
 *   O1 oracle_knn          brute-force exact kNN, fp32 d2 in the fixed FMA order,
 *                          keys (bits(d2) << 32 | j) ascending -- "finding
 *                          corresponding points".
 *   O2 oracle_covariance   fp64 mean / scatter (1/k), cyclic Jacobi eigen, GICP
 *                          plane regularisation C = V diag(eps,1,1) V^T -- the
 *                          Gaussian model p_i ~ N(p_i, C_i) with
 *                          "computing covariance ... C^p_i and C^q_i" (l.404).
 *   O3 oracle_linearize    d_i = q_i - T p_i (eq_trans_err, l.382-387), Mahalanobis
 *                          cost d^T (C^q + R C^p R^T)^-1 d (eq_trans_err_dist /
 *                          eq_trans_likelihood, l.388-402, read with the plus sign
 *                          and the inverse -- DESIGN.md readings R1/R2), J for the
 *                          left perturbation T <- Exp(delta) T, Neumaier sums.
 *   O4 oracle_align        host Levenberg-Marquardt on O3 (T = argmin ..., l.396-402).
 *   O5 oracle_kernel_eval  Table I kernel descriptors (l.420-435), written out.
 *   O7 oracle_linearize_vgicp / O8 oracle_align_vgicp  voxelized GICP (l.419):
 *                          voxel N, mean, mean covariance; pairs with the voxels
 *                          around fl32(T p); N-weighted Mahalanobis terms.
 *   O11 oracle_submap_query  sliding-window submap: the points of the arc-length
 *                          buckets around a pose (l.477-481).
 *   O10 oracle_cluster     Euclidean cluster extraction (l.549-559): connected
 *                          components under d2 <= tol^2, brute-force union-find.
 *   O9 oracle_ground_filter  z-vote ground filter: 2-D cell counts, keep cells
 *                          with >= min_count points (l.500-520).
 *   O6 oracle_covariance_kd  kernel-weighted mean / scatter + PLANE / MIN_EIG /
 *                          NORMALIZED_MIN_EIG regularisation (SURVEY §8(f) #1,
 *                          "covariance computation using the kernel descriptors" l.413).
 *
 * Parity status: every function here is pinned by tests/test_oracle_*.py against
 * closed forms, LAPACK, an fp32-FMA emulation, finite differences and known
 * transforms (see DESIGN.md §Oracle pins). No function is "parity unpinned".
 *
 * Build: gcc -O2 -ffp-contract=off -fopenmp -fPIC -shared (no -ffast-math).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_OK 0
#define ORACLE_EINVAL -1
#define ORACLE_EK -2
#define ORACLE_EDEGENERATE -6

#define LIN_REUSE_CORR 1

/* ------------------------------------------------------------------------- */
/* O1: fp32 squared distance in the fixed order                               */
/*   dx = qx - px; dy = qy - py; dz = qz - pz;                                */
/*   d2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx))                                 */
/* (reading R9.)                                 */
/* Two builds of the same function: hardware FMA when the host has it, else   */
/* libm fmaf (correctly rounded either way).                                  */
/* ------------------------------------------------------------------------- */
__attribute__((target("fma"))) static inline float d2_fma_hw(const float* q, const float* p) {
    float dx = q[0] - p[0];
    float dy = q[1] - p[1];
    float dz = q[2] - p[2];
    return __builtin_fmaf(dz, dz, __builtin_fmaf(dy, dy, dx * dx));
}

static inline float d2_fma_sw(const float* q, const float* p) {
    float dx = q[0] - p[0];
    float dy = q[1] - p[1];
    float dz = q[2] - p[2];
    return fmaf(dz, dz, fmaf(dy, dy, dx * dx));
}

static inline uint64_t make_key(float d2, int64_t j) {
    uint32_t bits;
    memcpy(&bits, &d2, 4);
    return ((uint64_t)bits << 32) | (uint64_t)(uint32_t)j;
}

static int all_finite(const float* x, int64_t n3) {
    for (int64_t i = 0; i < n3; ++i)
        if (!isfinite(x[i])) return 0;
    return 1;
}

/* the k smallest keys of query i, ascending, by insertion into a sorted list */
__attribute__((target("fma"))) static void knn_one_hw(const float* tgt, int64_t n, const float* q, int k,
                                                      uint64_t* keys) {
    int filled = 0;
    for (int64_t j = 0; j < n; ++j) {
        uint64_t key = make_key(d2_fma_hw(q, tgt + 3 * j), j);
        if (filled == k && key >= keys[k - 1]) continue;
        int r = (filled < k) ? filled++ : k - 1;
        while (r > 0 && keys[r - 1] > key) {
            keys[r] = keys[r - 1];
            --r;
        }
        keys[r] = key;
    }
}

static void knn_one_sw(const float* tgt, int64_t n, const float* q, int k, uint64_t* keys) {
    int filled = 0;
    for (int64_t j = 0; j < n; ++j) {
        uint64_t key = make_key(d2_fma_sw(q, tgt + 3 * j), j);
        if (filled == k && key >= keys[k - 1]) continue;
        int r = (filled < k) ? filled++ : k - 1;
        while (r > 0 && keys[r - 1] > key) {
            keys[r] = keys[r - 1];
            --r;
        }
        keys[r] = key;
    }
}

static int have_fma(void) {
    __builtin_cpu_init();
    return __builtin_cpu_supports("fma");
}

int oracle_has_hw_fma(void) { return have_fma(); }

/* O1: nbr[i][r] = j, d2[i][r] = d2_ij for the k smallest (d2, j) keys. */
int oracle_knn(const float* tgt, int64_t n, const float* q, int64_t m, int k, int32_t* nbr, float* d2,
               int nthreads) {
    if (!tgt || !q || !nbr || !d2 || n <= 0 || m < 0) return ORACLE_EINVAL;
    if (k < 1 || k > 32 || k > n) return ORACLE_EK;
    if (!all_finite(tgt, 3 * n) || !all_finite(q, 3 * m)) return ORACLE_EINVAL;
    const int hw = have_fma();
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t i = 0; i < m; ++i) {
        uint64_t keys[32];
        if (hw)
            knn_one_hw(tgt, n, q + 3 * i, k, keys);
        else
            knn_one_sw(tgt, n, q + 3 * i, k, keys);
        for (int r = 0; r < k; ++r) {
            uint32_t bits = (uint32_t)(keys[r] >> 32);
            float f;
            memcpy(&f, &bits, 4);
            nbr[i * k + r] = (int32_t)(uint32_t)(keys[r] & 0xffffffffu);
            d2[i * k + r] = f;
        }
    }
    return ORACLE_OK;
}

/* the fp32 d2 of O1, exposed for tests */
float oracle_d2(const float q[3], const float p[3]) { return have_fma() ? d2_fma_hw(q, p) : d2_fma_sw(q, p); }

/* ------------------------------------------------------------------------- */
/* O2: symmetric 3x3 eigen by cyclic Jacobi (fp64)                             */
/* ------------------------------------------------------------------------- */

/* S given as full 3x3 row-major; lam ascending; V columns are eigenvectors. */
int oracle_jacobi3(const double S_in[9], double lam[3], double V[9]) {
    double a[3][3], v[3][3];
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
            a[r][c] = S_in[3 * r + c];
            v[r][c] = (r == c) ? 1.0 : 0.0;
        }
    double fro = 0.0;
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) fro += a[r][c] * a[r][c];
    fro = sqrt(fro);
    for (int sweep = 0; sweep < 64; ++sweep) {
        double off = sqrt(2.0 * (a[0][1] * a[0][1] + a[0][2] * a[0][2] + a[1][2] * a[1][2]));
        if (off <= 1e-15 * fro || off == 0.0) break;
        for (int p = 0; p < 2; ++p) {
            for (int qq = p + 1; qq < 3; ++qq) {
                if (a[p][qq] == 0.0) continue;
                /* classic Jacobi rotation annihilating a[p][q] */
                double theta = (a[qq][qq] - a[p][p]) / (2.0 * a[p][qq]);
                double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
                double c = 1.0 / sqrt(t * t + 1.0);
                double s = t * c;
                for (int r = 0; r < 3; ++r) { /* A <- A J */
                    double arp = a[r][p], arq = a[r][qq];
                    a[r][p] = c * arp - s * arq;
                    a[r][qq] = s * arp + c * arq;
                }
                for (int r = 0; r < 3; ++r) { /* A <- J^T A */
                    double apr = a[p][r], aqr = a[qq][r];
                    a[p][r] = c * apr - s * aqr;
                    a[qq][r] = s * apr + c * aqr;
                }
                for (int r = 0; r < 3; ++r) { /* V <- V J */
                    double vrp = v[r][p], vrq = v[r][qq];
                    v[r][p] = c * vrp - s * vrq;
                    v[r][qq] = s * vrp + c * vrq;
                }
            }
        }
    }
    /* sort ascending (selection sort on 3) */
    int idx[3] = {0, 1, 2};
    double d[3] = {a[0][0], a[1][1], a[2][2]};
    for (int i = 0; i < 2; ++i)
        for (int j = i + 1; j < 3; ++j)
            if (d[idx[j]] < d[idx[i]]) {
                int t = idx[i];
                idx[i] = idx[j];
                idx[j] = t;
            }
    for (int c = 0; c < 3; ++c) {
        lam[c] = d[idx[c]];
        for (int r = 0; r < 3; ++r) V[3 * r + c] = v[r][idx[c]];
    }
    return ORACLE_OK;
}

/* O2: cov[i] = (xx, xy, xz, yy, yz, zz) of V diag(eps,1,1) V^T; gap[i] =
 * (lam2 - lam1)/lam3 (0 when lam3 == 0); S6[i] = the raw scatter (nullable). */
int oracle_covariance(const float* xyz, int64_t n, const int32_t* nbr, int64_t m, int k, double eps,
                      double* cov, double* gap, double* S6, int nthreads) {
    if (!xyz || !nbr || !cov || n <= 0 || m < 0) return ORACLE_EINVAL;
    if (k < 1 || k > 32 || k > n) return ORACLE_EK;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
    int bad = 0;
#pragma omp parallel for schedule(static) reduction(| : bad)
    for (int64_t i = 0; i < m; ++i) {
        double X[32][3];
        for (int j = 0; j < k; ++j) {
            int32_t id = nbr[i * k + j];
            if (id < 0 || id >= n) {
                bad = 1;
                id = 0;
            }
            for (int a = 0; a < 3; ++a) X[j][a] = (double)xyz[3 * (int64_t)id + a];
        }
        double mu[3] = {0, 0, 0};
        for (int j = 0; j < k; ++j)
            for (int a = 0; a < 3; ++a) mu[a] += X[j][a];
        for (int a = 0; a < 3; ++a) mu[a] /= (double)k;
        double S[9] = {0};
        for (int j = 0; j < k; ++j)
            for (int a = 0; a < 3; ++a)
                for (int b = 0; b < 3; ++b) S[3 * a + b] += (X[j][a] - mu[a]) * (X[j][b] - mu[b]);
        for (int a = 0; a < 9; ++a) S[a] /= (double)k;
        double lam[3], V[9];
        oracle_jacobi3(S, lam, V);
        double C[9];
        if (lam[2] == 0.0) {
            /* all k neighbours identical: n = +z (reading R11) */
            double nz[3] = {0, 0, 1};
            for (int a = 0; a < 3; ++a)
                for (int b = 0; b < 3; ++b) C[3 * a + b] = (a == b ? 1.0 : 0.0) - (1.0 - eps) * nz[a] * nz[b];
        } else {
            double w[3] = {eps, 1.0, 1.0};
            for (int a = 0; a < 3; ++a)
                for (int b = 0; b < 3; ++b) {
                    double s = 0.0;
                    for (int c = 0; c < 3; ++c) s += V[3 * a + c] * w[c] * V[3 * b + c];
                    C[3 * a + b] = s;
                }
        }
        double* o = cov + 6 * i;
        o[0] = C[0];
        o[1] = C[1];
        o[2] = C[2];
        o[3] = C[4];
        o[4] = C[5];
        o[5] = C[8];
        if (gap) gap[i] = (lam[2] == 0.0) ? 0.0 : (lam[1] - lam[0]) / lam[2];
        if (S6) {
            double* s6 = S6 + 6 * i;
            s6[0] = S[0];
            s6[1] = S[1];
            s6[2] = S[2];
            s6[3] = S[4];
            s6[4] = S[5];
            s6[5] = S[8];
        }
    }
    return bad ? ORACLE_EINVAL : ORACLE_OK;
}

/* -------------------------------------------------------------------------- */
/* O5: kernel descriptors (Table I, l.420-435)     */
/* -------------------------------------------------------------------------- */

/* Table I, written out (readings R19-R21):
 *   RBF         exp(-||x - y||^2 * sigma)       (verbatim: times sigma)
 *   Gaussian    exp(-||x - y||^2 / (2 sigma^2))
 *   Polynomial  (alpha <x, y> + c)^d
 *   HI          sum_i min(x_i, y_i) / sum_i x_i  (x, y non-negative)
 *   Laplacian   exp(-||x - y|| / sigma)
 * kind 0 = uniform (weight 1). x is the query point, y the neighbour. */
enum { KD_UNIFORM = 0, KD_RBF = 1, KD_GAUSSIAN = 2, KD_POLYNOMIAL = 3, KD_HI = 4, KD_LAPLACIAN = 5 };

double oracle_kernel_eval(int kind, double sigma, double alpha, double c, int d, const double* x, const double* y) {
    double d2 = 0.0, dot = 0.0, smin = 0.0, sx = 0.0;
    for (int a = 0; a < 3; ++a) {
        d2 += (x[a] - y[a]) * (x[a] - y[a]);
        dot += x[a] * y[a];
        smin += x[a] < y[a] ? x[a] : y[a];
        sx += x[a];
    }
    switch (kind) {
        case KD_UNIFORM: return 1.0;
        case KD_RBF: return exp(-d2 * sigma);
        case KD_GAUSSIAN: return exp(-d2 / (2.0 * sigma * sigma));
        case KD_POLYNOMIAL: return pow(alpha * dot + c, (double)d);
        case KD_HI: return sx > 0.0 ? smin / sx : 1.0;
        case KD_LAPLACIAN: return exp(-sqrt(d2) / sigma);
        default: return NAN;
    }
}

/* O6: kernel-weighted covariance with a choice of regularisation.
 *   w_j = max(0, K(q_i - o, x_j - o)), HI on max(0, .) components (R20);
 *   all w_j == 0 -> uniform weights (R19);
 *   mu = sum w x / sum w, S = sum w (x - mu)(x - mu)^T / sum w   (R19);
 *   reg 0 PLANE: V diag(eps,1,1) V^T (lam3 == 0 -> n = +z, R11)
 *   reg 1 MIN_EIG: V diag(max(lam_i, eps)) V^T
 *   reg 2 NORMALIZED_MIN_EIG: V diag(max(lam_i / lam3, eps)) V^T (lam3 == 0 -> eps I)  (R21)
 * q = NULL uses xyz[i] as the query of row i (m <= n). */
int oracle_covariance_kd(const float* xyz, int64_t n, const float* q, const int32_t* nbr, int64_t m, int k, int kind,
                         double sigma, double alpha, double c, int degree, const double* origin, int reg, double eps,
                         double* cov, double* gap, int nthreads) {
    if (!xyz || !nbr || !cov || n <= 0 || m < 0 || (!q && m > n)) return ORACLE_EINVAL;
    if (k < 1 || k > 32 || k > n) return ORACLE_EK;
    if (kind < 0 || kind > 5 || reg < 0 || reg > 2) return ORACLE_EINVAL;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
    const double o[3] = {origin ? origin[0] : 0.0, origin ? origin[1] : 0.0, origin ? origin[2] : 0.0};
    int bad = 0;
#pragma omp parallel for schedule(static) reduction(| : bad)
    for (int64_t i = 0; i < m; ++i) {
        double X[32][3], w[32];
        const float* qi = q ? q + 3 * i : xyz + 3 * i;
        double Q[3];
        for (int a = 0; a < 3; ++a) {
            Q[a] = (double)qi[a] - o[a];
            if (kind == KD_HI && Q[a] < 0.0) Q[a] = 0.0;
        }
        double W = 0.0;
        for (int j = 0; j < k; ++j) {
            int32_t id = nbr[i * k + j];
            if (id < 0 || id >= n) {
                bad = 1;
                id = 0;
            }
            double Y[3];
            for (int a = 0; a < 3; ++a) {
                X[j][a] = (double)xyz[3 * (int64_t)id + a];
                Y[a] = X[j][a] - o[a];
                if (kind == KD_HI && Y[a] < 0.0) Y[a] = 0.0;
            }
            double wj = oracle_kernel_eval(kind, sigma, alpha, c, degree, Q, Y);
            if (!(wj > 0.0)) wj = 0.0; /* also NaN */
            w[j] = wj;
            W += wj;
        }
        if (!(W > 0.0)) {
            for (int j = 0; j < k; ++j) w[j] = 1.0;
            W = (double)k;
        }
        double mu[3] = {0, 0, 0};
        for (int j = 0; j < k; ++j)
            for (int a = 0; a < 3; ++a) mu[a] += w[j] * X[j][a];
        for (int a = 0; a < 3; ++a) mu[a] /= W;
        double S[9] = {0};
        for (int j = 0; j < k; ++j)
            for (int a = 0; a < 3; ++a)
                for (int b = 0; b < 3; ++b) S[3 * a + b] += w[j] * (X[j][a] - mu[a]) * (X[j][b] - mu[b]);
        for (int a = 0; a < 9; ++a) S[a] /= W;
        double lam[3], V[9];
        oracle_jacobi3(S, lam, V);
        double lw[3];
        int eye = 0;
        if (reg == 0) {
            if (lam[2] == 0.0) { /* S = 0: n = +z (R11); columns (0,0,1), (0,1,0), (1,0,0) */
                const double P[9] = {0, 0, 1, 0, 1, 0, 1, 0, 0};
                for (int a = 0; a < 9; ++a) V[a] = P[a];
            }
            lw[0] = eps;
            lw[1] = 1.0;
            lw[2] = 1.0;
        } else if (reg == 1) {
            for (int a = 0; a < 3; ++a) lw[a] = lam[a] > eps ? lam[a] : eps;
        } else {
            if (lam[2] > 0.0) {
                for (int a = 0; a < 3; ++a) lw[a] = lam[a] / lam[2] > eps ? lam[a] / lam[2] : eps;
            } else {
                eye = 1;
            }
        }
        double C[9];
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) {
                double s = 0.0;
                if (eye) {
                    s = (a == b) ? eps : 0.0;
                } else {
                    for (int cc = 0; cc < 3; ++cc) s += V[3 * a + cc] * lw[cc] * V[3 * b + cc];
                }
                C[3 * a + b] = s;
            }
        double* out = cov + 6 * i;
        out[0] = C[0];
        out[1] = C[1];
        out[2] = C[2];
        out[3] = C[4];
        out[4] = C[5];
        out[5] = C[8];
        if (gap) gap[i] = (lam[2] == 0.0) ? 0.0 : (lam[1] - lam[0]) / lam[2];
    }
    return bad ? ORACLE_EINVAL : ORACLE_OK;
}

/* ------------------------------------------------------------------------- */
/* O3: linearize                                                              */
/* ------------------------------------------------------------------------- */

/* Cholesky inverse of a 3x3 SPD matrix (full row-major in, full out). */
static int spd_inverse3(const double A[9], double Minv[9]) {
    double L[3][3] = {{0}};
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j <= i; ++j) {
            double s = A[3 * i + j];
            for (int p = 0; p < j; ++p) s -= L[i][p] * L[j][p];
            if (i == j) {
                if (!(s > 0.0)) return -1;
                L[i][i] = sqrt(s);
            } else {
                L[i][j] = s / L[j][j];
            }
        }
    /* solve A x = e_c for each column c */
    for (int c = 0; c < 3; ++c) {
        double y[3], x[3];
        for (int i = 0; i < 3; ++i) {
            double s = (i == c) ? 1.0 : 0.0;
            for (int p = 0; p < i; ++p) s -= L[i][p] * y[p];
            y[i] = s / L[i][i];
        }
        for (int i = 2; i >= 0; --i) {
            double s = y[i];
            for (int p = i + 1; p < 3; ++p) s -= L[p][i] * x[p];
            x[i] = s / L[i][i];
        }
        for (int i = 0; i < 3; ++i) Minv[3 * i + c] = x[i];
    }
    return 0;
}

static void cov6_to_full(const float* c6, double C[9]) {
    C[0] = c6[0];
    C[1] = c6[1];
    C[2] = c6[2];
    C[3] = c6[1];
    C[4] = c6[3];
    C[5] = c6[4];
    C[6] = c6[2];
    C[7] = c6[4];
    C[8] = c6[5];
}

typedef struct {
    double s, c;
} neumaier;

static inline void nm_add(neumaier* a, double x) {
    double t = a->s + x;
    if (fabs(a->s) >= fabs(x))
        a->c += (a->s - t) + x;
    else
        a->c += (x - t) + a->s;
    a->s = t;
}

/* per-point term of one inlier: H (21 upper, row-major), b (6), e.
 * J = [skew(p' - c) | -I3] for the pivoted left perturbation
 * T <- Tr(c) Exp(delta) Tr(-c) T (reading R13); H = J^T M J;
 * b = J^T M d; e = d^T M d. */
static void point_terms(const double pp_in[3], const double c[3], const double d[3], const double M[9],
                        double out[28]) {
    const double pp[3] = {pp_in[0] - c[0], pp_in[1] - c[1], pp_in[2] - c[2]};
    double J[3][6];
    /* skew(p' - c) = [[0,-z,y],[z,0,-x],[-y,x,0]] */
    J[0][0] = 0.0;
    J[0][1] = -pp[2];
    J[0][2] = pp[1];
    J[1][0] = pp[2];
    J[1][1] = 0.0;
    J[1][2] = -pp[0];
    J[2][0] = -pp[1];
    J[2][1] = pp[0];
    J[2][2] = 0.0;
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) J[r][3 + c] = (r == c) ? -1.0 : 0.0;
    double MJ[3][6];
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 6; ++c) {
            double s = 0.0;
            for (int p = 0; p < 3; ++p) s += M[3 * r + p] * J[p][c];
            MJ[r][c] = s;
        }
    int o = 0;
    for (int a = 0; a < 6; ++a)
        for (int b = a; b < 6; ++b) {
            double s = 0.0;
            for (int p = 0; p < 3; ++p) s += J[p][a] * MJ[p][b];
            out[o++] = s;
        }
    double Md[3];
    for (int r = 0; r < 3; ++r) Md[r] = M[3 * r + 0] * d[0] + M[3 * r + 1] * d[1] + M[3 * r + 2] * d[2];
    for (int a = 0; a < 6; ++a) out[21 + a] = J[0][a] * Md[0] + J[1][a] * Md[1] + J[2][a] * Md[2];
    out[27] = d[0] * Md[0] + d[1] * Md[1] + d[2] * Md[2];
}

/* brute-force 1-NN of s over all targets: smallest (d2, j) key */
__attribute__((target("fma"))) static int64_t nn_hw(const float* tgt, int64_t nt, const float s[3], float* best) {
    uint64_t bk = UINT64_MAX;
    for (int64_t j = 0; j < nt; ++j) {
        uint64_t key = make_key(d2_fma_hw(s, tgt + 3 * j), j);
        if (key < bk) bk = key;
    }
    uint32_t bits = (uint32_t)(bk >> 32);
    memcpy(best, &bits, 4);
    return (int64_t)(bk & 0xffffffffu);
}

static int64_t nn_sw(const float* tgt, int64_t nt, const float s[3], float* best) {
    uint64_t bk = UINT64_MAX;
    for (int64_t j = 0; j < nt; ++j) {
        uint64_t key = make_key(d2_fma_sw(s, tgt + 3 * j), j);
        if (key < bk) bk = key;
    }
    uint32_t bits = (uint32_t)(bk >> 32);
    memcpy(best, &bits, 4);
    return (int64_t)(bk & 0xffffffffu);
}

/* O3. out29 = H(21 upper row-major), b(6), e, n_inliers. absum29 (nullable) =
 * sum of |term| per component (the tolerance scale). corr (nullable unless
 * REUSE_CORR) = j* or -1. */
int oracle_linearize(const float* src, const float* src_cov, int64_t ns, const float* tgt, const float* tgt_cov,
                     int64_t nt, const double T[16], const double* pivot, float max_corr_dist, int flags,
                     double* out29, double* absum29, int32_t* corr, int nthreads) {
    const double c0[3] = {pivot ? pivot[0] : 0.0, pivot ? pivot[1] : 0.0, pivot ? pivot[2] : 0.0};
    if (!src || !src_cov || !tgt || !tgt_cov || !T || !out29 || ns < 0 || nt <= 0) return ORACLE_EINVAL;
    if ((flags & LIN_REUSE_CORR) && !corr) return ORACLE_EINVAL;
    if (!(max_corr_dist > 0.0f)) return ORACLE_EINVAL;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
    const int hw = have_fma();
    const float r2 = max_corr_dist * max_corr_dist; /* fp32 product */
    const double R[9] = {T[0], T[1], T[2], T[4], T[5], T[6], T[8], T[9], T[10]};
    const double t[3] = {T[3], T[7], T[11]};

    /* correspondence search is independent per point (parallel); the sums run
     * serially in input order afterwards */
    int32_t* cj = (int32_t*)malloc(sizeof(int32_t) * (ns > 0 ? ns : 1));
    if (!cj) return ORACLE_EINVAL;
    if (flags & LIN_REUSE_CORR) {
        for (int64_t i = 0; i < ns; ++i) cj[i] = corr[i];
    } else {
#pragma omp parallel for schedule(dynamic, 16)
        for (int64_t i = 0; i < ns; ++i) {
            double p[3] = {src[3 * i], src[3 * i + 1], src[3 * i + 2]};
            double pp[3];
            for (int a = 0; a < 3; ++a)
                pp[a] = fma(R[3 * a + 2], p[2], fma(R[3 * a + 1], p[1], fma(R[3 * a + 0], p[0], t[a])));
            float s[3] = {(float)pp[0], (float)pp[1], (float)pp[2]};
            float best;
            int64_t j = hw ? nn_hw(tgt, nt, s, &best) : nn_sw(tgt, nt, s, &best);
            cj[i] = (best < r2) ? (int32_t)j : -1;
        }
    }
    neumaier acc[28];
    double ab[28];
    memset(acc, 0, sizeof(acc));
    memset(ab, 0, sizeof(ab));
    int64_t ninl = 0;
    int bad = 0;
    for (int64_t i = 0; i < ns; ++i) {
        int32_t j = cj[i];
        if (j < 0) continue;
        if (j >= nt) {
            bad = 1;
            continue;
        }
        double p[3] = {src[3 * i], src[3 * i + 1], src[3 * i + 2]};
        double pp[3];
        for (int a = 0; a < 3; ++a)
            pp[a] = fma(R[3 * a + 2], p[2], fma(R[3 * a + 1], p[1], fma(R[3 * a + 0], p[0], t[a])));
        double q[3] = {tgt[3 * (int64_t)j], tgt[3 * (int64_t)j + 1], tgt[3 * (int64_t)j + 2]};
        double d[3] = {q[0] - pp[0], q[1] - pp[1], q[2] - pp[2]};
        double Cq[9], Cp[9], RC[9], A[9], M[9];
        cov6_to_full(tgt_cov + 6 * (int64_t)j, Cq);
        cov6_to_full(src_cov + 6 * i, Cp);
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) {
                double s = 0.0;
                for (int c = 0; c < 3; ++c) s += R[3 * a + c] * Cp[3 * c + b];
                RC[3 * a + b] = s;
            }
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) {
                double s = 0.0;
                for (int c = 0; c < 3; ++c) s += RC[3 * a + c] * R[3 * b + c];
                A[3 * a + b] = Cq[3 * a + b] + s;
            }
        if (spd_inverse3(A, M) != 0) {
            bad = 1;
            continue;
        }
        double term[28];
        point_terms(pp, c0, d, M, term);
        for (int c = 0; c < 28; ++c) {
            nm_add(&acc[c], term[c]);
            ab[c] += fabs(term[c]);
        }
        ++ninl;
    }
    for (int c = 0; c < 28; ++c) out29[c] = acc[c].s + acc[c].c;
    out29[28] = (double)ninl;
    if (absum29) {
        for (int c = 0; c < 28; ++c) absum29[c] = ab[c];
        absum29[28] = (double)ninl;
    }
    if (corr && !(flags & LIN_REUSE_CORR))
        for (int64_t i = 0; i < ns; ++i) corr[i] = cj[i];
    free(cj);
    return bad ? ORACLE_EINVAL : ORACLE_OK;
}

/* ------------------------------------------------------------------------- */
/* O4: SE(3) exponential and LM align                                          */
/* ------------------------------------------------------------------------- */

/* delta = (omega, v). T row-major 4x4. */
void oracle_se3_exp(const double delta[6], double T[16]) {
    const double w[3] = {delta[0], delta[1], delta[2]};
    const double v[3] = {delta[3], delta[4], delta[5]};
    double W[9] = {0, -w[2], w[1], w[2], 0, -w[0], -w[1], w[0], 0};
    double W2[9];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) {
            double s = 0;
            for (int c = 0; c < 3; ++c) s += W[3 * a + c] * W[3 * c + b];
            W2[3 * a + b] = s;
        }
    double th = sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
    double R[9], V[9];
    if (th < 1e-10) {
        for (int a = 0; a < 9; ++a) {
            R[a] = ((a % 4) == 0 ? 1.0 : 0.0) + W[a];
            V[a] = ((a % 4) == 0 ? 1.0 : 0.0);
        }
    } else {
        double A = sin(th) / th;
        double B = (1.0 - cos(th)) / (th * th);
        double C = (th - sin(th)) / (th * th * th);
        for (int a = 0; a < 9; ++a) {
            double I = ((a % 4) == 0 ? 1.0 : 0.0);
            R[a] = I + A * W[a] + B * W2[a];
            V[a] = I + B * W[a] + C * W2[a];
        }
    }
    memset(T, 0, 16 * sizeof(double));
    for (int a = 0; a < 3; ++a) {
        for (int b = 0; b < 3; ++b) T[4 * a + b] = R[3 * a + b];
        T[4 * a + 3] = V[3 * a + 0] * v[0] + V[3 * a + 1] * v[1] + V[3 * a + 2] * v[2];
    }
    T[15] = 1.0;
}

static void mat4_mul(const double A[16], const double B[16], double C[16]) {
    double t[16];
    for (int a = 0; a < 4; ++a)
        for (int b = 0; b < 4; ++b) {
            double s = 0;
            for (int c = 0; c < 4; ++c) s += A[4 * a + c] * B[4 * c + b];
            t[4 * a + b] = s;
        }
    memcpy(C, t, sizeof(t));
}

/* Tr(c) Exp(delta) Tr(-c): rotation about the pivot c (reading R13) */
void oracle_pivoted_exp(const double delta[6], const double c[3], double T[16]) {
    double E[16];
    oracle_se3_exp(delta, E);
    memcpy(T, E, sizeof(E));
    for (int a = 0; a < 3; ++a) {
        double rc = E[4 * a + 0] * c[0] + E[4 * a + 1] * c[1] + E[4 * a + 2] * c[2];
        T[4 * a + 3] = E[4 * a + 3] + c[a] - rc;
    }
}
#define pivoted_exp oracle_pivoted_exp

/* solve (A) x = y for 6x6 SPD A by LDL^T (no pivoting). returns -1 if not PD */
int oracle_ldlt_solve6(const double A[36], const double y[6], double x[6]) {
    double L[6][6] = {{0}}, D[6];
    for (int j = 0; j < 6; ++j) {
        double s = A[6 * j + j];
        for (int p = 0; p < j; ++p) s -= L[j][p] * L[j][p] * D[p];
        D[j] = s;
        if (!(s > 0.0)) return -1;
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
        z[i] = s;
    }
    for (int i = 0; i < 6; ++i) z[i] /= D[i];
    for (int i = 5; i >= 0; --i) {
        double s = z[i];
        for (int p = i + 1; p < 6; ++p) s -= L[p][i] * x[p];
        x[i] = s;
    }
    return 0;
}

typedef struct {
    int max_iter;
    int lm;
    double rot_eps;
    double trans_eps;
    float max_corr_dist;
} oracle_align_params;

typedef struct {
    double T[16];
    int iterations;
    int converged;
    double error;
    int64_t inliers;
} oracle_align_result;

static void unpack_H(const double* o29, double H[36], double b[6]) {
    int o = 0;
    for (int a = 0; a < 6; ++a)
        for (int c = a; c < 6; ++c) {
            H[6 * a + c] = o29[o];
            H[6 * c + a] = o29[o];
            ++o;
        }
    for (int a = 0; a < 6; ++a) b[a] = o29[21 + a];
}

/* One record per LM trial (test instrumentation: recorded, never read back here).
 * [0] outer iteration, [1] lambda of the trial, [2] e at T, [3] e' at the trial pose,
 * [4] rho, [5] accepted, [6..11] delta, [12..17] b, [18..38] H (upper 21). */
#define ORACLE_TRACE_W 40
static void trace_put(double* tr, int cap, int* nt, int it, double lambda, double e, double en, double rho,
                      int acc, const double delta[6], const double* o29) {
    if (!tr || *nt >= cap) return;
    double* r = tr + (int64_t)ORACLE_TRACE_W * (*nt);
    r[0] = it;
    r[1] = lambda;
    r[2] = e;
    r[3] = en;
    r[4] = rho;
    r[5] = acc;
    for (int a = 0; a < 6; ++a) r[6 + a] = delta[a];
    for (int a = 0; a < 6; ++a) r[12 + a] = o29[21 + a];
    for (int a = 0; a < 21; ++a) r[18 + a] = o29[a];
    r[39] = 0.0;
    ++*nt;
}

/* O4: LM (lm=1) or Gauss-Newton (lm=0: lambda = 0, every step accepted).
 * oracle_align_ex additionally records every LM trial into trace[cap][40] (may be NULL). */
int oracle_align_ex(const float* src, const float* src_cov, int64_t ns, const float* tgt, const float* tgt_cov,
                    int64_t nt, const double T0[16], const oracle_align_params* prm, oracle_align_result* res,
                    int nthreads, double* trace, int trace_cap, int* n_trace) {
    int ntr = 0;
    if (!prm || !res || !T0) return ORACLE_EINVAL;
    double T[16];
    memcpy(T, T0, sizeof(T));
    int32_t* corr = (int32_t*)malloc(sizeof(int32_t) * (ns > 0 ? ns : 1));
    if (!corr) return ORACLE_EINVAL;
    double lambda = -1.0, nu = 2.0;
    int converged = 0, it = 0, rc = ORACLE_OK;
    double err = 0.0;
    int64_t inl = 0;
    for (it = 1; it <= prm->max_iter; ++it) {
        double o29[29];
        /* pivot: the source frame origin in the target frame (the sensor) */
        const double piv[3] = {T[3], T[7], T[11]};
        rc = oracle_linearize(src, src_cov, ns, tgt, tgt_cov, nt, T, piv, prm->max_corr_dist, 0, o29, NULL, corr,
                              nthreads);
        if (rc != ORACLE_OK) break;
        inl = (int64_t)o29[28];
        if (inl < 6) {
            rc = ORACLE_EDEGENERATE;
            break;
        }
        double H[36], b[6], delta[6] = {0};
        unpack_H(o29, H, b);
        double e = o29[27];
        err = e;
        if (!prm->lm) {
            double nb[6];
            for (int a = 0; a < 6; ++a) nb[a] = -b[a];
            if (oracle_ldlt_solve6(H, nb, delta) != 0) {
                rc = ORACLE_EDEGENERATE;
                break;
            }
            double dT[16];
            pivoted_exp(delta, piv, dT);
            mat4_mul(dT, T, T);
        } else {
            if (lambda < 0) {
                double mx = 0;
                for (int a = 0; a < 6; ++a)
                    if (H[7 * a] > mx) mx = H[7 * a];
                lambda = 1e-9 * mx;
            }
            int accepted = 0;
            for (int inner = 0; inner < 10; ++inner) {
                double Hl[36], nb[6];
                memcpy(Hl, H, sizeof(Hl));
                for (int a = 0; a < 6; ++a) {
                    Hl[7 * a] += lambda;
                    nb[a] = -b[a];
                }
                if (oracle_ldlt_solve6(Hl, nb, delta) != 0) {
                    lambda *= nu;
                    nu *= 2.0;
                    continue;
                }
                double dT[16], Tn[16];
                pivoted_exp(delta, piv, dT);
                mat4_mul(dT, T, Tn);
                double o2[29];
                rc = oracle_linearize(src, src_cov, ns, tgt, tgt_cov, nt, Tn, piv, prm->max_corr_dist,
                                      LIN_REUSE_CORR, o2, NULL, corr, nthreads);
                if (rc != ORACLE_OK) break;
                double en = o2[27];
                double den = 0.0;
                for (int a = 0; a < 6; ++a) den += delta[a] * (lambda * delta[a] - b[a]);
                double rho = (e - en) / den;
                trace_put(trace, trace_cap, &ntr, it, lambda, e, en, rho, rho > 0, delta, o29);
                if (rho > 0) {
                    memcpy(T, Tn, sizeof(T));
                    double f = 1.0 - pow(2.0 * rho - 1.0, 3);
                    lambda *= (f > 1.0 / 3.0) ? f : 1.0 / 3.0;
                    nu = 2.0;
                    err = en;
                    accepted = 1;
                    break;
                }
                lambda *= nu;
                nu *= 2.0;
            }
            if (rc != ORACLE_OK) break;
            if (!accepted) {
                /* no step decreases the cost: a (numerical) minimum */
                converged = 1;
                break;
            }
        }
        double mw = fmax(fabs(delta[0]), fmax(fabs(delta[1]), fabs(delta[2])));
        double mv = fmax(fabs(delta[3]), fmax(fabs(delta[4]), fabs(delta[5])));
        if (mw < prm->rot_eps && mv < prm->trans_eps) {
            converged = 1;
            break;
        }
    }
    free(corr);
    memcpy(res->T, T, sizeof(T));
    res->iterations = (it > prm->max_iter) ? prm->max_iter : it;
    res->converged = converged;
    res->error = err;
    res->inliers = inl;
    if (n_trace) *n_trace = ntr;
    return rc;
}

int oracle_align(const float* src, const float* src_cov, int64_t ns, const float* tgt, const float* tgt_cov,
                 int64_t nt, const double T0[16], const oracle_align_params* prm, oracle_align_result* res,
                 int nthreads) {
    return oracle_align_ex(src, src_cov, ns, tgt, tgt_cov, nt, T0, prm, res, nthreads, NULL, 0, NULL);
}

/* -------------------------------------------------------------------------- */
/* O7/O8: voxelized GICP ("extends and optimizes the Voxelized-  */
/* GICP"; readings R22-R23)                       */
/* -------------------------------------------------------------------------- */

/* voxel of a point: c_a = floor(fl32(fl32(x_a - o_a) * fl32(1/res))), o = the
 * target's per-axis minimum (the index's grid). */
static void vox_coord(const float* x, const float o[3], float inv, int64_t c[3]) {
    for (int a = 0; a < 3; ++a) {
        volatile float d = x[a] - o[a];
        volatile float t = d * inv;
        c[a] = (int64_t)floor((double)t);
    }
}

typedef struct {
    int64_t c[3];
    int64_t idx; /* target point */
} vox_item;

static int vox_cmp(const void* pa, const void* pb) {
    const vox_item* a = (const vox_item*)pa;
    const vox_item* b = (const vox_item*)pb;
    for (int k = 0; k < 3; ++k) {
        if (a->c[k] < b->c[k]) return -1;
        if (a->c[k] > b->c[k]) return 1;
    }
    return (a->idx < b->idx) ? -1 : (a->idx > b->idx);
}

typedef struct {
    int64_t c[3];
    int64_t n;
    double mu[3];
    double S[9]; /* mean of the points' covariances */
} voxel;

static int vcmp_key(const int64_t c[3], const voxel* v) {
    for (int k = 0; k < 3; ++k) {
        if (c[k] < v->c[k]) return -1;
        if (c[k] > v->c[k]) return 1;
    }
    return 0;
}

/* voxel statistics of the target (R22): N, mu = sum x / N, Sigma = sum C_j / N */
static voxel* build_voxels(const float* tgt, const float* tgt_cov, int64_t nt, float res, float o[3], float* inv,
                           int64_t* nv) {
    for (int a = 0; a < 3; ++a) {
        o[a] = tgt[a];
        for (int64_t j = 1; j < nt; ++j)
            if (tgt[3 * j + a] < o[a]) o[a] = tgt[3 * j + a];
    }
    volatile float iv = 1.0f / res;
    *inv = iv;
    vox_item* it = (vox_item*)malloc(sizeof(vox_item) * nt);
    voxel* vs = (voxel*)malloc(sizeof(voxel) * nt);
    if (!it || !vs) {
        free(it);
        free(vs);
        return NULL;
    }
    for (int64_t j = 0; j < nt; ++j) {
        vox_coord(tgt + 3 * j, o, *inv, it[j].c);
        it[j].idx = j;
    }
    qsort(it, nt, sizeof(vox_item), vox_cmp);
    int64_t m = 0;
    for (int64_t s = 0; s < nt;) {
        int64_t e = s;
        while (e < nt && it[e].c[0] == it[s].c[0] && it[e].c[1] == it[s].c[1] && it[e].c[2] == it[s].c[2]) ++e;
        voxel* v = &vs[m++];
        for (int a = 0; a < 3; ++a) v->c[a] = it[s].c[a];
        v->n = e - s;
        double mu[3] = {0, 0, 0}, S[9] = {0};
        for (int64_t r = s; r < e; ++r) {
            const int64_t j = it[r].idx;
            double C[9];
            cov6_to_full(tgt_cov + 6 * j, C);
            for (int a = 0; a < 3; ++a) mu[a] += (double)tgt[3 * j + a];
            for (int a = 0; a < 9; ++a) S[a] += C[a];
        }
        for (int a = 0; a < 3; ++a) v->mu[a] = mu[a] / (double)v->n;
        for (int a = 0; a < 9; ++a) v->S[a] = S[a] / (double)v->n;
        s = e;
    }
    free(it);
    *nv = m;
    return vs;
}

static const voxel* find_voxel(const voxel* vs, int64_t nv, const int64_t c[3]) {
    int64_t lo = 0, hi = nv - 1;
    while (lo <= hi) {
        const int64_t mid = (lo + hi) / 2;
        const int r = vcmp_key(c, &vs[mid]);
        if (r == 0) return &vs[mid];
        if (r < 0)
            hi = mid - 1;
        else
            lo = mid + 1;
    }
    return NULL;
}

/* neighbour sets: own voxel, + 6 faces, + 12 edges + 8 corners (nearest-first) */
static const int vg_off[27][3] = {{0, 0, 0},   {-1, 0, 0},  {1, 0, 0},   {0, -1, 0},  {0, 1, 0},   {0, 0, -1},
                                  {0, 0, 1},   {-1, -1, 0}, {1, -1, 0},  {-1, 1, 0},  {1, 1, 0},   {-1, 0, -1},
                                  {1, 0, -1},  {-1, 0, 1},  {1, 0, 1},   {0, -1, -1}, {0, 1, -1},  {0, -1, 1},
                                  {0, 1, 1},   {-1, -1, -1}, {1, -1, -1}, {-1, 1, -1}, {1, 1, -1}, {-1, -1, 1},
                                  {1, -1, 1},  {-1, 1, 1},  {1, 1, 1}};

/* O7: out29 = sum over (source i, voxel v in the neighbour set of fl32(T p_i)) of
 * (with LIN_REUSE_CORR the base voxel of each i is taken from base[3i..] -- the
 * previous linearisation's -- instead of fl32(T p_i); otherwise it is written there) 
 * N_v * (J^T M J, J^T M d, d^T M d) with d = mu_v - T p_i, M = (Sigma_v + R C_i
 * R^T)^-1, J about the pivot; out29[28] = number of pairs. Neumaier sums in
 * (i, offset) order; absum29 = sum |term|. mode = 1, 7 or 27. */
int oracle_linearize_vgicp(const float* src, const float* src_cov, int64_t ns, const float* tgt,
                           const float* tgt_cov, int64_t nt, float res, const double T[16], const double* pivot,
                           int mode, int flags, int32_t* base, double* out29, double* absum29) {
    if (!src || !src_cov || !tgt || !tgt_cov || !T || !out29 || ns < 0 || nt <= 0 || !(res > 0.0f)) return ORACLE_EINVAL;
    if ((flags & LIN_REUSE_CORR) && !base) return ORACLE_EINVAL;
    if (mode != 1 && mode != 7 && mode != 27) return ORACLE_EINVAL;
    const double c0[3] = {pivot ? pivot[0] : 0.0, pivot ? pivot[1] : 0.0, pivot ? pivot[2] : 0.0};
    float o[3], inv;
    int64_t nv = 0;
    voxel* vs = build_voxels(tgt, tgt_cov, nt, res, o, &inv, &nv);
    if (!vs) return ORACLE_EINVAL;
    const double R[9] = {T[0], T[1], T[2], T[4], T[5], T[6], T[8], T[9], T[10]};
    const double t[3] = {T[3], T[7], T[11]};
    neumaier acc[28];
    double ab[28];
    memset(acc, 0, sizeof(acc));
    memset(ab, 0, sizeof(ab));
    int64_t pairs = 0;
    int bad = 0;
    for (int64_t i = 0; i < ns; ++i) {
        const double p[3] = {src[3 * i], src[3 * i + 1], src[3 * i + 2]};
        double pp[3];
        for (int a = 0; a < 3; ++a) pp[a] = fma(R[3 * a + 2], p[2], fma(R[3 * a + 1], p[1], fma(R[3 * a + 0], p[0], t[a])));
        const float s[3] = {(float)pp[0], (float)pp[1], (float)pp[2]};
        int64_t c[3];
        if (flags & LIN_REUSE_CORR) { /* the pairs of the previous linearisation (R23) */
            for (int a = 0; a < 3; ++a) c[a] = base[3 * i + a];
        } else {
            vox_coord(s, o, inv, c);
            if (base)
                for (int a = 0; a < 3; ++a) base[3 * i + a] = (int32_t)c[a];
        }
        double Cp[9], RC[9], RCR[9];
        cov6_to_full(src_cov + 6 * i, Cp);
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) {
                double v = 0.0;
                for (int k = 0; k < 3; ++k) v += R[3 * a + k] * Cp[3 * k + b];
                RC[3 * a + b] = v;
            }
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) {
                double v = 0.0;
                for (int k = 0; k < 3; ++k) v += RC[3 * a + k] * R[3 * b + k];
                RCR[3 * a + b] = v;
            }
        for (int u = 0; u < mode; ++u) {
            const int64_t cn[3] = {c[0] + vg_off[u][0], c[1] + vg_off[u][1], c[2] + vg_off[u][2]};
            const voxel* v = find_voxel(vs, nv, cn);
            if (!v) continue;
            double A[9], M[9];
            for (int a = 0; a < 9; ++a) A[a] = v->S[a] + RCR[a];
            if (spd_inverse3(A, M) != 0) {
                bad = 1;
                continue;
            }
            const double d[3] = {v->mu[0] - pp[0], v->mu[1] - pp[1], v->mu[2] - pp[2]};
            double term[28];
            point_terms(pp, c0, d, M, term);
            for (int k = 0; k < 28; ++k) {
                const double w = (double)v->n * term[k];
                nm_add(&acc[k], w);
                ab[k] += fabs(w);
            }
            ++pairs;
        }
    }
    for (int k = 0; k < 28; ++k) out29[k] = acc[k].s + acc[k].c;
    out29[28] = (double)pairs;
    if (absum29) {
        for (int k = 0; k < 28; ++k) absum29[k] = ab[k];
        absum29[28] = (double)pairs;
    }
    free(vs);
    return bad ? ORACLE_EINVAL : ORACLE_OK;
}

/* O8: LM on O7 with R13's schedule; the trial cost e' keeps the pairs of the
 * linearisation (the base voxels, R23), as gicp_align keeps its correspondences. */
int oracle_align_vgicp(const float* src, const float* src_cov, int64_t ns, const float* tgt, const float* tgt_cov,
                       int64_t nt, float res, int mode, const double T0[16], const oracle_align_params* prm,
                       oracle_align_result* out) {
    if (!prm || !out || !T0) return ORACLE_EINVAL;
    double T[16];
    memcpy(T, T0, sizeof(T));
    double lambda = -1.0, nu = 2.0, err = 0.0;
    int converged = 0, it = 0, rc = ORACLE_OK;
    int64_t inl = 0;
    int32_t* base = (int32_t*)malloc(sizeof(int32_t) * 3 * (ns > 0 ? ns : 1));
    if (!base) return ORACLE_EINVAL;
    for (it = 1; it <= prm->max_iter; ++it) {
        double o29[29];
        const double piv[3] = {T[3], T[7], T[11]};
        rc = oracle_linearize_vgicp(src, src_cov, ns, tgt, tgt_cov, nt, res, T, piv, mode, 0, base, o29, NULL);
        if (rc != ORACLE_OK) break;
        inl = (int64_t)o29[28];
        if (inl < 6) {
            rc = ORACLE_EDEGENERATE;
            break;
        }
        double H[36], b[6], delta[6] = {0};
        unpack_H(o29, H, b);
        const double e = o29[27];
        err = e;
        if (lambda < 0) {
            double mx = 0;
            for (int a = 0; a < 6; ++a)
                if (H[7 * a] > mx) mx = H[7 * a];
            lambda = 1e-9 * mx;
        }
        int accepted = 0;
        for (int inner = 0; inner < 10; ++inner) {
            double Hl[36], nb[6];
            memcpy(Hl, H, sizeof(Hl));
            for (int a = 0; a < 6; ++a) {
                Hl[7 * a] += lambda;
                nb[a] = -b[a];
            }
            if (oracle_ldlt_solve6(Hl, nb, delta) != 0) {
                lambda *= nu;
                nu *= 2.0;
                continue;
            }
            double dT[16], Tn[16], o2[29];
            oracle_pivoted_exp(delta, piv, dT);
            mat4_mul(dT, T, Tn);
            const double pn[3] = {Tn[3], Tn[7], Tn[11]};
            rc = oracle_linearize_vgicp(src, src_cov, ns, tgt, tgt_cov, nt, res, Tn, pn, mode, LIN_REUSE_CORR, base, o2,
                                        NULL);
            if (rc != ORACLE_OK) break;
            const double en = o2[27];
            double den = 0.0;
            for (int a = 0; a < 6; ++a) den += delta[a] * (lambda * delta[a] - b[a]);
            const double rho = (e - en) / den;
            if (rho > 0) {
                memcpy(T, Tn, sizeof(T));
                const double f = 1.0 - pow(2.0 * rho - 1.0, 3);
                lambda *= (f > 1.0 / 3.0) ? f : 1.0 / 3.0;
                nu = 2.0;
                err = en;
                accepted = 1;
                break;
            }
            lambda *= nu;
            nu *= 2.0;
        }
        if (rc != ORACLE_OK) break;
        if (!accepted) {
            converged = 1;
            break;
        }
        const double mw = fmax(fabs(delta[0]), fmax(fabs(delta[1]), fabs(delta[2])));
        const double mv = fmax(fabs(delta[3]), fmax(fabs(delta[4]), fabs(delta[5])));
        if (mw < prm->rot_eps && mv < prm->trans_eps) {
            converged = 1;
            break;
        }
    }
    free(base);
    memcpy(out->T, T, sizeof(T));
    out->iterations = (it > prm->max_iter) ? prm->max_iter : it;
    out->converged = converged;
    out->error = err;
    out->inliers = inl;
    return rc;
}

/* -------------------------------------------------------------------------- */
/* O9: z-vote ground filter ("vote the points corresponding  */
/* to the grid-cell ... filter out ground points ... without matrix computation"; */
/* SURVEY.md §8(f) #4; reading R24)                   */
/* -------------------------------------------------------------------------- */

/* cell (u, v) = (floor(fl32(x * fl32(1/cell))), floor(fl32(y * fl32(1/cell)))) in
 * the points' (vehicle body) frame; count[i] = the number of points in i's cell;
 * keep[i] = count[i] >= min_count (a vertical feature). */
typedef struct {
    int64_t u, v, i;
} uv_item;

static int uv_cmp(const void* pa, const void* pb) {
    const uv_item* a = (const uv_item*)pa;
    const uv_item* b = (const uv_item*)pb;
    if (a->u != b->u) return a->u < b->u ? -1 : 1;
    if (a->v != b->v) return a->v < b->v ? -1 : 1;
    return (a->i < b->i) ? -1 : (a->i > b->i);
}

int oracle_ground_filter(const float* xyz, int64_t n, float cell, int min_count, int32_t* count, uint8_t* keep) {
    if (!xyz || n < 0 || !(cell > 0.0f) || !keep) return ORACLE_EINVAL;
    if (n == 0) return ORACLE_OK;
    volatile float iv = 1.0f / cell;
    const float inv = iv;
    uv_item* it = (uv_item*)malloc(sizeof(uv_item) * n);
    if (!it) return ORACLE_EINVAL;
    for (int64_t i = 0; i < n; ++i) {
        volatile float tu = xyz[3 * i] * inv, tv = xyz[3 * i + 1] * inv;
        it[i].u = (int64_t)floor((double)tu);
        it[i].v = (int64_t)floor((double)tv);
        it[i].i = i;
    }
    qsort(it, n, sizeof(uv_item), uv_cmp);
    for (int64_t s = 0; s < n;) {
        int64_t e = s;
        while (e < n && it[e].u == it[s].u && it[e].v == it[s].v) ++e;
        for (int64_t r = s; r < e; ++r) {
            if (count) count[it[r].i] = (int32_t)(e - s);
            keep[it[r].i] = (e - s) >= min_count;
        }
        s = e;
    }
    free(it);
    return ORACLE_OK;
}

/* -------------------------------------------------------------------------- */
/* O10: Euclidean cluster extraction ("CUDA-based Euclidean   */
/* distance clustering ... to find cluster C_j" citing Rusu 2010       */
/* §8(f) #4; reading R25)                              */
/* -------------------------------------------------------------------------- */

static int64_t uf_find(int64_t* p, int64_t x) {
    while (p[x] != x) {
        p[x] = p[p[x]];
        x = p[x];
    }
    return x;
}

/* i ~ j iff d2(p_i, p_j) <= fl32(tol * tol) with the R9 fp32 d2; clusters = the
 * connected components; those with fewer than min_size points get label -1;
 * the rest are numbered 0, 1, ... by descending size, ties by the smallest
 * member index. O(n^2) pairs (brute force). Returns the number of clusters. */
int64_t oracle_cluster(const float* xyz, int64_t n, float tol, int min_size, int32_t* label) {
    if (!xyz || n < 0 || !(tol > 0.0f) || !label) return -1;
    if (n == 0) return 0;
    const int hw = have_fma();
    const float t2 = tol * tol;
    int64_t* par = (int64_t*)malloc(sizeof(int64_t) * n);
    if (!par) return -1;
    for (int64_t i = 0; i < n; ++i) par[i] = i;
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = i + 1; j < n; ++j) {
            const float d2 = hw ? d2_fma_hw(xyz + 3 * i, xyz + 3 * j) : d2_fma_sw(xyz + 3 * i, xyz + 3 * j);
            if (d2 <= t2) {
                const int64_t a = uf_find(par, i), b = uf_find(par, j);
                if (a != b) par[a > b ? a : b] = a < b ? a : b;
            }
        }
    /* component of each point = its root (the smallest member index) */
    int64_t* size = (int64_t*)calloc(n, sizeof(int64_t));
    if (!size) {
        free(par);
        return -1;
    }
    for (int64_t i = 0; i < n; ++i) size[uf_find(par, i)]++;
    int64_t nc = 0;
    for (int64_t r = 0; r < n; ++r)
        if (size[r] >= min_size && size[r] > 0) ++nc;
    int64_t* roots = (int64_t*)malloc(sizeof(int64_t) * (nc > 0 ? nc : 1));
    int64_t* rank = (int64_t*)malloc(sizeof(int64_t) * n);
    if (!roots || !rank) {
        free(par); free(size); free(roots); free(rank);
        return -1;
    }
    int64_t k = 0;
    for (int64_t r = 0; r < n; ++r)
        if (size[r] >= min_size && size[r] > 0) roots[k++] = r;
    /* insertion sort by (size desc, root asc) -- roots ascending already */
    for (int64_t a = 1; a < nc; ++a) {
        const int64_t x = roots[a];
        int64_t b = a - 1;
        while (b >= 0 && size[roots[b]] < size[x]) {
            roots[b + 1] = roots[b];
            --b;
        }
        roots[b + 1] = x;
    }
    for (int64_t r = 0; r < n; ++r) rank[r] = -1;
    for (int64_t a = 0; a < nc; ++a) rank[roots[a]] = a;
    for (int64_t i = 0; i < n; ++i) label[i] = (int32_t)rank[uf_find(par, i)];
    free(par); free(size); free(roots); free(rank);
    return nc;
}

/* -------------------------------------------------------------------------- */
/* O11: sliding-window submap query ("associate each pose on  */
/* the race line with its corresponding point cloud map" via a GPU hash; "points  */
/* from M_i^psi instead of the entire unified map"; DESIGN R26)   */
/* -------------------------------------------------------------------------- */

/* points of the buckets center - radius .. center + radius (mod n_buckets, each
 * bucket once; radius >= n_buckets / 2 covers the whole track), in window order
 * (center - radius first), original order inside a bucket. Returns the count. */
int64_t oracle_submap_query(const int32_t* bucket, int64_t n, int n_buckets, int center, int radius, int32_t* out) {
    if (!bucket || n < 0 || n_buckets < 1 || radius < 0 || center < 0 || center >= n_buckets) return -1;
    int64_t span = 2 * (int64_t)radius + 1;
    if (span > n_buckets) span = n_buckets;
    int64_t m = 0;
    for (int64_t w = 0; w < span; ++w) {
        const int b = (int)((((int64_t)center - radius + w) % n_buckets + n_buckets) % n_buckets);
        for (int64_t i = 0; i < n; ++i)
            if (bucket[i] == b) out[m++] = (int32_t)i;
    }
    return m;
}
