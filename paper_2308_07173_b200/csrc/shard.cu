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

// table[gid[e]] = rows[e] for the entries launched this round (poses[e].active)
__global__ void k_scatter_rows(const double* __restrict__ rows, int E, const int* __restrict__ gid,
                               const Pose* __restrict__ poses, double* __restrict__ table) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= (int64_t)E * 32) return;
    const int e = (int)(i >> 5), c = (int)(i & 31);
    if (poses && !poses[e].active) return;
    table[(int64_t)gid[e] * 32 + c] = rows[i];
}

// out[b][c] = sum over chunks k = 0..nc-1, in that order, of table[b][k][c]; one
// block; then (optional) the host-mapped completion flag
__global__ void k_combine_chunks(const double* __restrict__ table, int B, int nc, int width, double* __restrict__ out,
                                 volatile unsigned* flag, unsigned seq) {
    for (int64_t i = threadIdx.x; i < (int64_t)B * width; i += blockDim.x) {
        const int64_t b = i / width;
        const int c = (int)(i % width);
        const double* t = table + (b * nc) * width + c;
        double v = 0.0;
        for (int k = 0; k < nc; ++k) v += t[(int64_t)k * width];
        out[i] = v;
    }
    if (flag) {
        __threadfence_system();
        __syncthreads();
        if (threadIdx.x == 0) *flag = seq;
    }
}

}  // namespace

int launch_scatter_rows(const double* rows, int E, const int* gid_dev, const Pose* poses_dev, double* table,
                        cudaStream_t s) {
    if (E <= 0) return GICP_OK;
    const int64_t n = (int64_t)E * 32;
    k_scatter_rows<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(rows, E, gid_dev, poses_dev, table);
    return check_cuda(cudaGetLastError(), "scatter rows");
}

int launch_combine_chunks(const double* table, int B, int nc, int width, double* out, volatile unsigned* flag,
                          unsigned seq, cudaStream_t s) {
    k_combine_chunks<<<1, 256, 0, s>>>(table, B, nc, width, out, flag, seq);
    return check_cuda(cudaGetLastError(), "combine chunks");
}

}  // namespace gicp
