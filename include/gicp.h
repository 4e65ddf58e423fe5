/*
 * gicp.h -- C ABI of the B200-native GICP hot path (libgicp_b200.so).
 *
 * The paper (arxiv 2308.07173, §III-C1 "Efficient registration method",
 * l.377-435) models scans P, Q as Gaussian clouds p_i ~ N(p_i, C^p_i) (l.380),
 * defines d_i = q_i - T p_i (eq_trans_err, l.382-387) and registers by
 * T = argmin sum_i d_i^T (C^q_i + R C^p_i R^T)^-1 d_i (eq_trans_likelihood,
 * l.396-402, read with '+' and the inverse: DESIGN.md readings R1/R2). Its GPU
 * contribution is "nearest points search and covariance computation" (l.413,
 * l.798) -- the calls below -- plus the per-iteration linearisation this build
 * adds.
 *
 * Conventions for every call:
 *  - Pointers are DEVICE pointers (CUDA global memory of the current device)
 *    unless marked (host). Point clouds are fp32 xyz, [n][3] row-major, 4-byte
 *    aligned. Covariances are fp32 [n][6] = (xx, xy, xz, yy, yz, zz).
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    knn / covariances / linearize are stream-ordered and asynchronous with
 *    respect to the host; build_index and align are synchronous.
 *  - Ownership: the caller owns every buffer it passes in and every output
 *    buffer; the library never frees them. An index owns a private device copy
 *    of its points (the caller may free xyz after gicp_build_index returns) plus
 *    scratch; it is immutable after build except for that scratch, so calls on
 *    one index must be serialised by the caller (one stream at a time).
 *  - Errors: argument errors are detected synchronously and returned as a
 *    negative code; gicp_last_error() gives a thread-local message. Kernel
 *    launch failures return GICP_ECUDA. Outputs never contain NaN for finite
 *    inputs.
 */
#ifndef GICP_B200_H
#define GICP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GICP_KMAX 32

enum {
    GICP_OK = 0,
    GICP_EINVAL = -1,      /* null pointer, n <= 0, bad cell size / radius, non-finite coordinates */
    GICP_EK = -2,          /* k < 1 || k > GICP_KMAX || k > n_target */
    GICP_ERANGE = -3,      /* the voxel grid would exceed 2^21 cells per axis */
    GICP_ENOMEM = -4,      /* device allocation failed */
    GICP_ECUDA = -5,       /* a CUDA runtime call or kernel launch failed */
    GICP_EDEGENERATE = -6  /* fewer than 6 gated correspondences */
};

typedef struct gicp_index_s* gicp_index;

/* Thread-local message describing the last failure of this thread ("" if none). */
const char* gicp_last_error(void);

/* Library ABI version (major * 100 + minor). */
int gicp_version(void);

/* ---------------------------------------------------------------------------
 * gicp_build_index -- the spatial structure behind "GPU-based nearest points
 * search" ("GPU-hash data structure", l.477): a uniform voxel
 * grid built by radix sort on (Morton) cell keys, plus coarser levels of the same
 * grid (cell x 2^l) that share the sorted points, used for queries whose
 * neighbourhood is wider than the base cell (sparse regions of a scan).
 *   xyz        [n][3] fp32 target cloud (device). Must be finite (checked).
 *   n          number of points, 1 <= n < 2^31.
 *   cell_size  voxel edge in metres (> 0), or 0 for an automatic choice
 *              (about 1.15 x the expected 20-NN radius, from the occupancy of a
 *              trial grid).
 *   out (host) receives the new index on success.
 * Synchronous (returns after the build completed on `stream`).
 * Errors: EINVAL (null, n <= 0, cell_size < 0 / non-finite, non-finite xyz),
 *         ERANGE (grid too fine for the bounding box), ENOMEM, ECUDA.
 * ------------------------------------------------------------------------- */
int gicp_build_index(const float* xyz, int64_t n, float cell_size, void* stream, gicp_index* out);

/* Releases the index and all device memory it owns. NULL is a no-op. */
void gicp_index_free(gicp_index idx);

typedef struct {
    int64_t n;            /* points */
    int64_t n_cells;      /* occupied voxels */
    float cell_size;      /* metres */
    float origin[3];      /* grid origin (bounding-box minimum) */
    int32_t dims[3];      /* voxels per axis (level 0) */
    int64_t device_bytes; /* device memory owned by the index */
    int32_t n_levels;     /* voxel pyramid levels (cell_l = cell_size * 2^l) */
} gicp_index_info;

/* Attach the covariances of the index's points (cov [n][6], ORIGINAL order,
 * device; e.g. the output of gicp_knn_cov_self): the index keeps a copy permuted
 * into its sorted order, and gicp_linearize / gicp_align use that copy whenever
 * they are passed this same `cov` pointer as tgt_cov (the results are identical;
 * the target covariance is then read next to the target point instead of by a
 * random gather). Re-attach after modifying `cov`. Stream-ordered.
 * Errors: EINVAL (null), ENOMEM, ECUDA. */
int gicp_index_attach_cov(gicp_index idx, const float* cov, void* stream);

/* Host-side description of an index. Errors: EINVAL. */
int gicp_get_index_info(gicp_index idx, gicp_index_info* info /* host */);

/* ---------------------------------------------------------------------------
 * gicp_knn -- exact k nearest neighbours of external queries ("finding
 * corresponding points"). For each query i, the k smallest
 * keys (d2, j) over ALL n target points, where
 *   dx = qx - px; dy = qy - py; dz = qz - pz;  d2 = fmaf(dz,dz, fmaf(dy,dy, dx*dx))
 * in fp32 round-to-nearest (reading R9), ties broken by the target's
 * ORIGINAL index j. Rows ascend by (d2, j).
 *   q      [m][3] fp32 queries (device); a non-finite query yields nbr = -1, d2 = +inf.
 *   nbr    [m][k] int32 out: original target indices.
 *   d2     [m][k] fp32 out: squared distances.
 * Errors: EINVAL (null, m < 0), EK. m = 0 is a no-op.
 * ------------------------------------------------------------------------- */
int gicp_knn(gicp_index idx, const float* q, int64_t m, int k, int32_t* nbr, float* d2, void* stream);

/* As gicp_knn with the index's own points as the queries, rows in the points'
 * original order (the query itself is its own first neighbour unless an exact
 * duplicate with a smaller index exists). nbr/d2 are [n][k]. */
int gicp_knn_self(gicp_index idx, int k, int32_t* nbr, float* d2, void* stream);

/* ---------------------------------------------------------------------------
 * gicp_covariances -- per-point covariance C_i for the Gaussian model (PAPER.md
 * l.380, l.404 "computing covariance when estimate the C^p_i and C^q_i"):
 *   mu = (1/k) sum_j x_nbr[i][j];  S = (1/k) sum_j (x - mu)(x - mu)^T;
 *   eigenvalues of S replaced by (eps, 1, 1) in ascending order (GICP plane
 *   regularisation, reading R7): C = I - (1 - eps) n n^T with n the
 *   smallest-eigenvalue eigenvector; n = +z when all k neighbours coincide (R11).
 *   xyz    [n][3] fp32 cloud that nbr indexes (device).
 *   nbr    [m][k] int32 (device), each in [0, n).
 *   eps    regularisation, 0 < eps <= 1 (1e-3 in GICP).
 *   cov    [m][6] fp32 out.
 * Errors: EINVAL (null, n <= 0, m < 0, eps out of range), EK. Out-of-range
 * nbr entries are a caller error (undefined results, no fault: clamped).
 * ------------------------------------------------------------------------- */
int gicp_covariances(const float* xyz, int64_t n, const int32_t* nbr, int64_t m, int k, float eps, float* cov,
                     void* stream);

/* Fused kNN + covariance over the index's own points in one kernel (the hot
 * path of the headline workload). Outputs as gicp_knn_self + gicp_covariances;
 * nbr and d2 may be NULL to skip writing them. */
int gicp_knn_cov_self(gicp_index idx, int k, float eps, int32_t* nbr, float* d2, float* cov, void* stream);

/* ---------------------------------------------------------------------------
 * gicp_covariances_kd -- kernel-descriptor weighted covariances (PAPER.md l.413
 * "covariance computation using the kernel descriptors", Table I l.420-435;
 * SURVEY.md §8(f) #1; readings R19-R21):
 *   w_j = max(0, K(q_i - o, x_j - o)) for the K of Table I (x = the query):
 *     RBF exp(-||x-y||^2 * sigma) (verbatim), Gaussian exp(-||x-y||^2/(2 sigma^2)),
 *     Polynomial (alpha <x,y> + c)^degree, HI sum min(x_i,y_i) / sum x_i on the
 *     non-negative parts, Laplacian exp(-||x-y||/sigma), or uniform;
 *   all weights 0 -> uniform; mu = sum w x / sum w; S = sum w (x-mu)(x-mu)^T / sum w;
 *   reg PLANE: V diag(eps,1,1) V^T (as gicp_covariances), MIN_EIG:
 *   V diag(max(lam, eps)) V^T, NORMALIZED_MIN_EIG: V diag(max(lam/lam_max, eps)) V^T.
 *   xyz [n][3] cloud the neighbours index, q [m][3] queries or NULL (row i's query
 *   is xyz[i], m <= n), nbr [m][k], cov [m][6] out (device). params (host).
 * Errors: EINVAL (null, n <= 0, m < 0, sigma <= 0 for the distance kernels,
 * degree < 1 or > 16 for Polynomial, eps out of (0, 1], unknown kind / reg), EK.
 * ------------------------------------------------------------------------- */
enum { GICP_KD_UNIFORM = 0, GICP_KD_RBF = 1, GICP_KD_GAUSSIAN = 2, GICP_KD_POLYNOMIAL = 3, GICP_KD_HI = 4,
       GICP_KD_LAPLACIAN = 5 };
enum { GICP_REG_PLANE = 0, GICP_REG_MIN_EIG = 1, GICP_REG_NORMALIZED_MIN_EIG = 2 };
typedef struct {
    int kernel;        /* GICP_KD_* */
    float sigma;       /* RBF / Gaussian / Laplacian */
    float alpha, c;    /* Polynomial */
    int degree;        /* Polynomial, 1..16 */
    float origin[3];   /* o: Polynomial / HI coordinates are x - o */
    int reg;           /* GICP_REG_* */
    float eps;         /* 1e-3 */
} gicp_cov_params;

int gicp_covariances_kd(const float* xyz, int64_t n, const float* q, const int32_t* nbr, int64_t m, int k,
                        const gicp_cov_params* params /* host */, float* cov, void* stream);

/* ---------------------------------------------------------------------------
 * gicp_linearize -- one GICP linearisation at pose T (PAPER.md eq_trans_err
 * l.382-387, eq_trans_likelihood l.396-402; readings R1-R4, R12):
 *   p'  = R p + t in fp64 (a-th row: fma(R_a2, p_z, fma(R_a1, p_y, fma(R_a0, p_x, t_a))))
 *   s   = fl32(p');  j* = argmin_j (d2(s, q_j), j) over ALL targets (d2 as gicp_knn)
 *   inlier iff d2 < fl32(r*r);   d = q_j* - p';  M = (C^q_j* + R C^p_i R^T)^-1
 *   J = [skew(p' - c) | -I3] for the perturbation T <- Tr(c) Exp(delta) Tr(-c) T,
 *   delta = (omega, v): a rotation about the pivot c, then a translation
 *   (reading R13; c = 0 is the plain left perturbation)
 *   out29 = sum over inliers of J^T M J (21 upper-triangle entries, row-major),
 *           J^T M d (6), d^T M d (1), inlier count (1)  -- fp64, deterministic
 *           fixed-order reduction (bitwise reproducible run to run).
 *   src, src_cov  [ns][3], [ns][6] fp32 (device).
 *   tgt           index built on the target cloud; tgt_cov [nt][6] fp32 in the
 *                 target's ORIGINAL order (device).
 *   T (host)      4x4 row-major fp64 (rigid).
 *   pivot (host)  fp64 [3] rotation pivot c in the target frame, or NULL for the
 *                 origin; gicp_align uses the source origin mapped by T (the
 *                 sensor), which keeps lever arms short in map coordinates.
 *   max_corr_dist gate r in metres (> 0).
 *   flags         GICP_LIN_REUSE_CORR: skip the search and use corr[] as given
 *                 (entries < 0 are outliers); GICP_LIN_ERROR_ONLY: only e and the
 *                 count are accumulated (H and b are written as 0).
 *   out29         device fp64 [29] out.
 *   corr          [ns] int32 out (j* or -1), nullable unless REUSE_CORR.
 * Errors: EINVAL (null, ns < 0, r <= 0), ENOMEM (scratch), ECUDA.
 * ------------------------------------------------------------------------- */
enum { GICP_LIN_REUSE_CORR = 1, GICP_LIN_ERROR_ONLY = 2 };

int gicp_linearize(const float* src, const float* src_cov, int64_t ns, gicp_index tgt, const float* tgt_cov,
                   const double T[16] /* host */, const double* pivot /* host, nullable */, float max_corr_dist,
                   int flags, double* out29, int32_t* corr, void* stream);

/* ---------------------------------------------------------------------------
 * gicp_align -- host Levenberg-Marquardt over gicp_linearize (T = argmin ...,
 * PAPER.md l.396-402; the optimiser is DESIGN.md reading R13):
 *   per iteration: pivot c = T's translation, linearize at T (search), lambda
 *   init 1e-9 max diag(H), up to 10 inner trials solving (H + lambda I) delta = -b
 *   (LDL^T), T' = Tr(c) Exp(delta) Tr(-c) T,
 *   e' = linearize(T', REUSE_CORR, ERROR_ONLY), gain rho = (e - e')/(delta^T
 *   (lambda delta - b)); accept iff rho > 0 (lambda *= max(1/3, 1 - (2 rho - 1)^3))
 *   else lambda *= nu, nu *= 2; converged when the ACCEPTED step has
 *   max|delta_omega| < rot_eps and max|delta_v| < trans_eps, or when no trial
 *   decreases the cost (a numerical minimum). lm = 0 gives plain Gauss-Newton.
 * Synchronous. Errors: EINVAL, EDEGENERATE (< 6 inliers), ENOMEM, ECUDA.
 * Non-convergence is not an error (result->converged = 0).
 * ------------------------------------------------------------------------- */
typedef struct {
    int max_iter;        /* 64 */
    int lm;              /* 1 = Levenberg-Marquardt, 0 = Gauss-Newton */
    double rot_eps;      /* 1e-6 rad */
    double trans_eps;    /* 1e-5 m */
    float max_corr_dist; /* 1.0 m */
} gicp_align_params;

typedef struct {
    double T[16];        /* final pose, row-major */
    int iterations;      /* outer iterations run */
    int converged;       /* 1 if the step criterion was met */
    double error;        /* cost at the final pose (last accepted evaluation) */
    int64_t inliers;     /* inliers of the last linearisation */
} gicp_align_result;

int gicp_align(const float* src, const float* src_cov, int64_t ns, gicp_index tgt, const float* tgt_cov,
               const double T0[16] /* host */, const gicp_align_params* params /* host */,
               gicp_align_result* result /* host */, void* stream);

/* ---------------------------------------------------------------------------
 * Batched registration (many scans against one map).
 * B registrations with concatenated sources: registration b owns source points
 * [offsets[b], offsets[b+1]) of src / src_cov (device) and corr; offsets is a
 * host int64 [B+1] array with offsets[0] = 0, non-decreasing.
 *
 * gicp_linearize_batched -- gicp_linearize for every registration in ONE launch:
 *   T (host) fp64 [B][16], pivots (host) fp64 [B][3] or NULL (origins),
 *   out29 (device) fp64 [B][29] (row b = registration b; zero for an empty
 *   one). Each registration is partitioned and reduced exactly as a single
 *   gicp_linearize over its own points, so row b is bitwise the single result.
 *   Flags and errors as gicp_linearize. Asynchronous (stream-ordered).
 *
 * gicp_align_batched -- gicp_align for every registration, in lockstep: each
 *   evaluation round (initial linearisation, LM trials, re-linearisation) is one
 *   batched launch over the registrations that need it. Per registration the
 *   iterates are those of gicp_align on it alone (bitwise). T0 (host) [B][16],
 *   result (host) [B]. A registration with < 6 correspondences stops (its
 *   result holds the last pose and inlier count) and the call returns
 *   GICP_EDEGENERATE after finishing the others. Synchronous.
 * ------------------------------------------------------------------------- */
int gicp_linearize_batched(const float* src, const float* src_cov, const int64_t* offsets /* host [B+1] */, int B,
                           gicp_index tgt, const float* tgt_cov, const double* T /* host [B][16] */,
                           const double* pivots /* host [B][3] or NULL */, float max_corr_dist, int flags,
                           double* out29 /* device [B][29] */, int32_t* corr, void* stream);

int gicp_align_batched(const float* src, const float* src_cov, const int64_t* offsets /* host [B+1] */, int B,
                       gicp_index tgt, const float* tgt_cov, const double* T0 /* host [B][16] */,
                       const gicp_align_params* params /* host */, gicp_align_result* result /* host [B] */,
                       void* stream);

/* gicp_align_batched_ex -- the sharded form: this process holds
 * E entries (point ranges offsets[E+1] of src), entry e belonging to
 * registration entry_reg[e] (host int [E], NULL = identity with E == B). After
 * every evaluation round the library calls
 *     reduce(entry_rows, E, reg_rows, B, user)
 * with entry_rows (host) [E][32] -- per entry: out29 (H 21, b 6, e, count), the
 * trial cost with the previous correspondences and its count, one pad -- and
 * the callback must fill reg_rows (host) [B][32] with the sum over ALL processes'
 * entries of each registration (a cross-rank allreduce; summing a fixed global
 * chunking in chunk order makes the result independent of the process count).
 * It returns 0 on success. Every process must run the same B registrations with
 * the same T0 and params: the host LM decisions depend on reg_rows only, so all
 * processes take the same rounds and their collectives stay matched. reduce =
 * NULL sums the local entries of each registration in entry order. */
typedef int (*gicp_reduce_fn)(const double* entry_rows, int E, double* reg_rows, int B, void* user);

int gicp_align_batched_ex(const float* src, const float* src_cov, const int64_t* offsets /* host [E+1] */, int E,
                          const int* entry_reg /* host [E] or NULL */, int B, gicp_index tgt, const float* tgt_cov,
                          const double* T0 /* host [B][16] */, const gicp_align_params* params /* host */,
                          gicp_align_result* result /* host [B] */, gicp_reduce_fn reduce, void* user, void* stream);

/* gicp_align_batched_sharded -- the sharded form with the reduction on the device
 * ("one NCCL allreduce of the 27-float H/b over NVLink per
 * iteration"; the paper's data parallelism over points).
 * This process holds E entries (point ranges offsets[E+1] of src); entry e is
 * chunk c of registration b and entry_chunk[e] (host) = b * num_chunks + c, the
 * chunking being FIXED globally (independent of the number of processes). After
 * every evaluation round the library zeroes `table` (device, caller-owned,
 * [B * num_chunks][32] doubles), writes each launched entry's row (H 21, b 6, e,
 * count, trial cost, its count, pad) at its chunk row, calls
 *     allreduce(table, B * num_chunks * 32, user, stream)
 * which must sum `table` over all processes IN PLACE, stream-ordered on `stream`
 * (e.g. ncclAllReduce on it; NULL: a single process), then sums each
 * registration's chunk rows in chunk order on the device. Every row has one
 * contributor, so the allreduce is exact and H, b, e are bitwise identical for
 * any process count; every process then runs the identical host LM (all take the
 * same rounds: the collectives stay matched; a process without entries passes
 * E = 0 and still takes part). Returns as gicp_align_batched; allreduce returning
 * non-zero -> GICP_ECUDA. Synchronous. */
typedef int (*gicp_allreduce_fn)(double* table, int64_t count, void* user, void* stream);

int gicp_align_batched_sharded(const float* src, const float* src_cov, const int64_t* offsets /* host [E+1] */,
                               int E, const int* entry_chunk /* host [E] */, int num_chunks, int B, gicp_index tgt,
                               const float* tgt_cov, const double* T0 /* host [B][16] */,
                               const gicp_align_params* params /* host */, gicp_align_result* result /* host [B] */,
                               double* table /* device [B * num_chunks][32] */, gicp_allreduce_fn allreduce,
                               void* user, void* stream);

/* gicp_combine_chunks -- out[b][c] = sum over k = 0 .. num_chunks-1 (in that order)
 * of table[b][k][c]; table (device) [B][num_chunks][width], out (device) [B][width].
 * The chunk-ordered sum of a sharded one-shot linearisation (after the caller's
 * allreduce of the chunk table). Stream-ordered. */
int gicp_combine_chunks(const double* table, int B, int num_chunks, int width, double* out, void* stream);


/* ---------------------------------------------------------------------------
 * Voxelized GICP ("extends and optimizes the Voxelized-GICP";
 * SURVEY.md §8(f) #2; readings R22-R23). Build the target index with
 * cell_size = the VGICP resolution, then attach the voxel Gaussians:
 *
 * gicp_index_attach_voxels -- per level-0 voxel v: N_v, mean mu_v (fp64 sums,
 *   stored as an fp32 offset from the voxel's first point) and Sigma_v = the
 *   mean of its points' covariances cov [n][6] (original order, device).
 *   Asynchronous. Errors: EINVAL, ENOMEM.
 * gicp_linearize_vgicp -- out29 = sum over pairs (source i, voxel v among the
 *   voxel of fl32(T p_i) and its 6 faces (mode 7) / 26 neighbours (mode 27) / none
 *   (mode 1)) of N_v (J^T M J, J^T M d, d^T M d), d = mu_v - T p_i (fp64),
 *   M = (Sigma_v + R C_i R^T)^-1, J about the pivot (as gicp_linearize);
 *   out29[28] = the number of pairs. base: each source point's base voxel
 *   (cx, cy, cz), written unless GICP_LIN_REUSE_CORR, which reuses it (the pairs
 *   of a previous linearisation); GICP_LIN_ERROR_ONLY as gicp_linearize. Async.
 * gicp_align_vgicp -- gicp_align's LM on gicp_linearize_vgicp; the trial cost
 *   keeps the pairs of the linearisation. Synchronous.
 *   EDEGENERATE: < 6 pairs.
 * ------------------------------------------------------------------------- */
int gicp_index_attach_voxels(gicp_index idx, const float* cov, void* stream);
int gicp_linearize_vgicp(const float* src, const float* src_cov, int64_t ns, gicp_index tgt,
                         const double T[16] /* host */, const double* pivot /* host [3] or NULL */, int mode,
                         int flags, int32_t* base /* device [ns][3], nullable unless REUSE_CORR */,
                         double* out29 /* device [29] */, void* stream);
int gicp_align_vgicp(const float* src, const float* src_cov, int64_t ns, gicp_index tgt, int mode,
                     const double T0[16] /* host */, const gicp_align_params* params /* host */,
                     gicp_align_result* result /* host */, void* stream);


/* ---------------------------------------------------------------------------
 * gicp_ground_filter -- the z-vote vertical-feature extractor (PAPER.md l.500-520,
 * "vote the points corresponding to the grid-cell ... hashing ... filter out
 * ground points without matrix computation"; R24):
 *   cell (u, v) = (floor(fl32(x * fl32(1/cell))), floor(fl32(y * fl32(1/cell))))
 *   in the points' (vehicle body) frame, |u|, |v| clamped below 2^31 - 1;
 *   keep[i] = 1 iff i's cell holds >= min_count points (a vertical feature:
 *   walls, posts), 0 for ground; count[i] (nullable) = that number.
 *   The input is expected voxel-filtered (leaf <= cell, SPEC pre).
 *   xyz [n][3] fp32, keep [n] uint8, count [n] int32 (device). Asynchronous.
 * Errors: EINVAL (n < 0, cell <= 0, null), ENOMEM.
 * ------------------------------------------------------------------------- */
int gicp_ground_filter(const float* xyz, int64_t n, float cell, int min_count, uint8_t* keep, int32_t* count,
                       void* stream);


/* ---------------------------------------------------------------------------
 * gicp_cluster -- Euclidean cluster extraction (the
 * "CUDA-based Euclidean distance clustering" of Rusu 2010; SPEC S:549-556;
 * DESIGN.md R25): i ~ j iff d2(p_i, p_j) <= fl32(tol*tol) (fp32 d2 as gicp_knn);
 * clusters = connected components, numbered 0, 1, ... by descending size, ties
 * by the smallest member index; components with fewer than min_size points get
 * label -1. xyz [n][3], label [n] int32 (device); *n_clusters (host) = the
 * number of numbered clusters. Synchronous. Errors: EINVAL, ENOMEM, ERANGE.
 * ------------------------------------------------------------------------- */
int gicp_cluster(const float* xyz, int64_t n, float tol, int min_size, int32_t* label, int64_t* n_clusters,
                 void* stream);


/* ---------------------------------------------------------------------------
 * Sliding-window submap (a GPU hash associating each pose on
 * the race line with its map points; "points from M_i^psi instead of the entire
 * unified map"; R26).
 * gicp_submap_build -- bucket (device int32 [n]): each map point's arc-length
 *   bucket in [0, n_buckets) (the caller's race-line parametrisation; the track
 *   is closed). One stable sort by bucket + the bucket start table (a perfect
 *   hash: bucket ids are dense). Synchronous. EINVAL on an id out of range.
 * gicp_submap_query -- the map point indices of the buckets center - radius ..
 *   center + radius (mod n_buckets, each bucket once: radius >= n_buckets / 2 is
 *   the whole map), in that order, original order inside a bucket, into out
 *   (device int32, capacity >= the count); *count (host). Stream-ordered.
 * ------------------------------------------------------------------------- */
typedef struct gicp_submap_s* gicp_submap;
int gicp_submap_build(const int32_t* bucket, int64_t n, int n_buckets, gicp_submap* out, void* stream);
int gicp_submap_query(gicp_submap sm, int center, int radius, int32_t* out, int64_t* count, void* stream);
void gicp_submap_free(gicp_submap sm);


/* ---------------------------------------------------------------------------
 * Query sharding of the external kNN (config C5 across GPUs, SURVEY.md §8(e):
 * "queries sharded by cell-sorted ranges, map replicated ... rank 0 builds and
 * ncclBroadcasts the sorted float4 + cell table").
 *
 * gicp_knn_query_order -- perm (device int32 [m]) = the queries in the order the
 *   index's voxel grid sorts them (the order gicp_knn processes them in; non-finite
 *   queries last). A rank takes a contiguous range of it.
 * gicp_knn_subset -- gicp_knn restricted to the queries ids (device int32 [n_ids],
 *   indices into q [m][3]); rows ids[t] of nbr / d2 ([m][k], device) are written,
 *   the others untouched. Rows are bitwise those of gicp_knn (the per-query result
 *   does not depend on the other queries).
 * gicp_index_export -- the index's metadata as an opaque host header
 *   (GICP_INDEX_HEADER_BYTES) and its device buffers (pointers and byte sizes,
 *   GICP_INDEX_MAX_BUFFERS; a NULL pointer / 0 bytes: absent). The buffers stay
 *   owned by the index. Attached covariances / voxel statistics are not exported.
 * gicp_index_import -- a new index (owning copies) from a header and device
 *   buffers laid out as exported (e.g. received by a broadcast); synchronous.
 * ------------------------------------------------------------------------- */
#define GICP_INDEX_HEADER_BYTES 4096
#define GICP_INDEX_MAX_BUFFERS 16
int gicp_knn_query_order(gicp_index idx, const float* q, int64_t m, int32_t* perm, void* stream);
int gicp_knn_subset(gicp_index idx, const float* q, int64_t m, const int32_t* ids, int64_t n_ids, int k, int32_t* nbr,
                    float* d2, void* stream);
int gicp_index_export(gicp_index idx, void* header /* host [GICP_INDEX_HEADER_BYTES] */,
                      void** buffers /* host [GICP_INDEX_MAX_BUFFERS] */, int64_t* bytes /* host [..] */,
                      int* n_buffers /* host */);
int gicp_index_import(const void* header /* host */, const void* const* buffers /* host array of device pointers */,
                      void* stream, gicp_index* out);

/* gicp_align_timing -- opt-in diagnostics (bench.py's roofline): while enabled,
 * gicp_align and the batched aligns record CUDA events on their stream around every
 * linearisation launch of the calling thread. The call returns, per kind ([0]
 * speculative dual launches, [1] full linearisations, [2] trial costs), the
 * accumulated device milliseconds, launch counts and source points linearised
 * (active registrations' points, summed over the launches), resets them, and sets
 * the enable flag. Host pointers ([3] each), nullable. */
int gicp_align_timing(int enable, double* ms, int64_t* launches, int64_t* points);

#ifdef __cplusplus
}
#endif
#endif /* GICP_B200_H */
