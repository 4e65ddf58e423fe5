// shard.cu -- the device side of the sharded (multi-GPU) linearisation
// (DESIGN.md §9).
//
// Source points of every registration are split into a FIXED global chunking
// (num_chunks chunks of whole linearize blocks, independent of the world size).
// Per evaluation round a rank holds the 32-value rows of its chunks (out29 +
// the trial cost and its count + pad). They are scattered into a device table
// [B * num_chunks][32] that is zero elsewhere; ONE in-place allreduce(sum) over
// the ranks (NCCL, by the caller's callback) fills every row from its single
// owner, exactly (x + 0 = x); the combine kernel then sums each registration's
// chunk rows in chunk order. H, b and e are therefore bitwise identical for any
// number of ranks, and every rank's host LM takes the same decisions.
#include "gicp_internal.cuh"

namespace gicp {
namespace {

// table[gid[e]] = rows[e] for the entries launched this round (their registration's
// pose active, the entry non-empty)
__global__ void k_scatter_rows(const double* __restrict__ rows, int E, const int* __restrict__ gid,
                               const int* __restrict__ ereg, const Pose* __restrict__ poses,
                               const int64_t* __restrict__ offs, double* __restrict__ table) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= (int64_t)E * 32) return;
    const int e = (int)(i >> 5), c = (int)(i & 31);
    if (poses && !poses[ereg ? ereg[e] : e].active) return;
    if (offs && offs[e + 1] == offs[e]) return;
    table[(int64_t)gid[e] * 32 + c] = rows[i];
}

// out[b][c] = sum over chunks k = 0..nc-1, in that order, of table[b][k][c]; one
// thread per output value (the chunk loads are independent: unrolled by 8)
__global__ void k_combine_chunks(const double* __restrict__ table, int B, int nc, int width,
                                 double* __restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= (int64_t)B * width) return;
    const int64_t b = i / width;
    const int c = (int)(i % width);
    const double* t = table + (b * nc) * width + c;
    double v = 0.0;
    int k = 0;
    for (; k + 8 <= nc; k += 8) {
        double x[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) x[u] = __ldcg(t + (int64_t)(k + u) * width);
#pragma unroll
        for (int u = 0; u < 8; ++u) v += x[u];
    }
    for (; k < nc; ++k) v += __ldcg(t + (int64_t)k * width);
    out[i] = v;
}

// the host-mapped completion flag, after the stream's previous work
__global__ void k_signal(volatile unsigned* flag, unsigned seq) {
    __threadfence_system();
    *flag = seq;
}

// compact block table: thread i finds its active entry (binary search over the
// compact starts) and copies that entry's block from the full table
__global__ void k_compact_btab(const int4* __restrict__ btab, const int2* __restrict__ clist, int nce, int total,
                               int4* __restrict__ ctab) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= total) return;
    int lo = 0, hi = nce - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (clist[mid].y <= i) lo = mid; else hi = mid - 1;
    }
    ctab[i] = btab[clist[lo].x + (i - clist[lo].y)];
}

}  // namespace

int launch_compact_btab(const int4* btab, const int2* clist, int nce, int total, int4* ctab, cudaStream_t s) {
    if (total <= 0) return GICP_OK;
    k_compact_btab<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(btab, clist, nce, total, ctab);
    return check_cuda(cudaGetLastError(), "compact block table");
}

int launch_scatter_rows(const double* rows, int E, const int* gid_dev, const int* ereg_dev, const Pose* poses_dev,
                        const int64_t* offs_dev, double* table, cudaStream_t s) {
    if (E <= 0) return GICP_OK;
    const int64_t n = (int64_t)E * 32;
    k_scatter_rows<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(rows, E, gid_dev, ereg_dev, poses_dev, offs_dev, table);
    return check_cuda(cudaGetLastError(), "scatter rows");
}

int launch_combine_chunks(const double* table, int B, int nc, int width, double* out, volatile unsigned* flag,
                          unsigned seq, cudaStream_t s) {
    const int64_t n = (int64_t)B * width;
    if (n > 0) k_combine_chunks<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(table, B, nc, width, out);
    if (flag) k_signal<<<1, 1, 0, s>>>(flag, seq);
    return check_cuda(cudaGetLastError(), "combine chunks");
}

}  // namespace gicp
