// sortnet.cuh -- compile-time comparator networks for register-resident top-k lists.
//
// All networks act on "wires" (array slots that the unrolled device code keeps in
// registers) and are generated as constexpr tables, so after unrolling every wire
// index is a compile-time constant. An op (a, b, kind) leaves min(w_a, w_b) in wire a
// and max in wire b; kind 1 computes only the min (wire b is dead afterwards), kind 2
// only the max (wire a is dead). Pruning keeps exactly the ops whose results reach
// the first NOUT outputs.
//
//  * sort_net<N, NOUT>       Batcher odd-even merge sort of N wires; afterwards wire i
//                            holds the i-th smallest for i < NOUT.
//  * merge_net<M, B, NOUT>   Batcher odd-even merge of two sorted runs, wires 0..M-1 and
//                            M..M+B-1; out[r] = the wire holding the r-th smallest.
//
// Plain C++ (host and device): tests/test_sortnet.py compiles this header with g++
// and checks every network on all 0-1 inputs (the 0-1 principle).
#pragma once

#if defined(__CUDACC__)
#define SORTNET_HD __host__ __device__
#else
#define SORTNET_HD
#endif

namespace gicp {
namespace net {

constexpr int kMaxOps = 1024;
constexpr int kMaxWires = 72;

struct Net {
    int n = 0;                 // ops
    unsigned char a[kMaxOps]{};
    unsigned char b[kMaxOps]{};
    unsigned char kind[kMaxOps]{};
    unsigned char out[kMaxWires]{};  // merge networks: wire of the r-th smallest
};

constexpr void add_op(Net& t, int a, int b) {
    t.a[t.n] = (unsigned char)a;
    t.b[t.n] = (unsigned char)b;
    t.kind[t.n] = 0;
    ++t.n;
}

// Batcher odd-even merge of two sorted wire lists A (m) and B (nb) into out (m + nb);
// works for any lengths (TAOCP 5.3.4). Returns m + nb.
constexpr int oe_merge(Net& t, const int* A, int m, const int* B, int nb, int* out) {
    if (m == 0) {
        for (int i = 0; i < nb; ++i) out[i] = B[i];
        return nb;
    }
    if (nb == 0) {
        for (int i = 0; i < m; ++i) out[i] = A[i];
        return m;
    }
    if (m == 1 && nb == 1) {
        add_op(t, A[0], B[0]);
        out[0] = A[0];
        out[1] = B[0];
        return 2;
    }
    int Ae[kMaxWires] = {}, Ao[kMaxWires] = {}, Be[kMaxWires] = {}, Bo[kMaxWires] = {};
    int ne = 0, no = 0, me = 0, mo = 0;
    for (int i = 0; i < m; ++i) {
        if (i % 2 == 0) Ae[ne++] = A[i];
        else Ao[no++] = A[i];
    }
    for (int i = 0; i < nb; ++i) {
        if (i % 2 == 0) Be[me++] = B[i];
        else Bo[mo++] = B[i];
    }
    int V[kMaxWires] = {}, W[kMaxWires] = {};
    const int nv = oe_merge(t, Ae, ne, Be, me, V);
    const int nw = oe_merge(t, Ao, no, Bo, mo, W);
    out[0] = V[0];
    int o = 1, i = 1, j = 0;
    while (i < nv && j < nw) {
        add_op(t, W[j], V[i]);
        out[o++] = W[j++];
        out[o++] = V[i++];
    }
    while (i < nv) out[o++] = V[i++];
    while (j < nw) out[o++] = W[j++];
    return o;
}

// Keep only the ops whose results can reach wires live at the end (live[w] = 1);
// one-sided ops where only the min or only the max is used afterwards.
constexpr Net prune(const Net& t, const bool* live_end) {
    bool live[kMaxWires] = {};
    for (int w = 0; w < kMaxWires; ++w) live[w] = live_end[w];
    bool keep[kMaxOps] = {};
    unsigned char kind[kMaxOps] = {};
    for (int k = t.n - 1; k >= 0; --k) {
        const int a = t.a[k], b = t.b[k];
        const bool la = live[a], lb = live[b];
        if (!la && !lb) continue;
        keep[k] = true;
        kind[k] = (la && lb) ? 0 : (la ? 1 : 2);
        live[a] = live[b] = true;
    }
    Net r{};
    for (int k = 0; k < t.n; ++k)
        if (keep[k]) {
            r.a[r.n] = t.a[k];
            r.b[r.n] = t.b[k];
            r.kind[r.n] = kind[k];
            ++r.n;
        }
    for (int w = 0; w < kMaxWires; ++w) r.out[w] = t.out[w];
    return r;
}

// sort N wires in place (merge sort by recursive halving), outputs 0..NOUT-1 live
constexpr int oe_sort(Net& t, const int* A, int n, int* out) {
    if (n <= 1) {
        for (int i = 0; i < n; ++i) out[i] = A[i];
        return n;
    }
    const int h = n / 2;
    int L[kMaxWires] = {}, R[kMaxWires] = {};
    oe_sort(t, A, h, L);
    oe_sort(t, A + h, n - h, R);
    return oe_merge(t, L, h, R, n - h, out);
}

template <int N, int NOUT>
constexpr Net make_sort_net() {
    static_assert(NOUT <= N && N <= kMaxWires, "sort_net: NOUT <= N");
    Net t{};
    int A[kMaxWires] = {}, out[kMaxWires] = {};
    for (int i = 0; i < N; ++i) A[i] = i;
    oe_sort(t, A, N, out);
    for (int i = 0; i < N; ++i) t.out[i] = (unsigned char)out[i];
    bool live[kMaxWires] = {};
    for (int i = 0; i < NOUT; ++i) live[out[i]] = true;
    return prune(t, live);
}

template <int M, int B, int NOUT>
constexpr Net make_merge_net() {
    static_assert(NOUT <= M + B && M + B <= kMaxWires, "merge_net: NOUT <= M + B");
    Net t{};
    int A[kMaxWires] = {}, Bw[kMaxWires] = {}, out[kMaxWires] = {};
    for (int i = 0; i < M; ++i) A[i] = i;
    for (int i = 0; i < B; ++i) Bw[i] = M + i;
    oe_merge(t, A, M, Bw, B, out);
    for (int i = 0; i < M + B; ++i) t.out[i] = (unsigned char)out[i];
    bool live[kMaxWires] = {};
    for (int i = 0; i < NOUT; ++i) live[out[i]] = true;
    return prune(t, live);
}

// Apply a constexpr network `t` (a constant expression in the caller) to a register
// array of unsigned keys: min/max are single instructions on 32-bit integers. A
// macro, so that every wire index stays a compile-time constant after unrolling.
#define GICP_APPLY_NET(v, t)                                          \
    _Pragma("unroll") for (int k_ = 0; k_ < (t).n; ++k_) {            \
        const unsigned x_ = (v)[(t).a[k_]], y_ = (v)[(t).b[k_]];      \
        if ((t).kind[k_] != 2) (v)[(t).a[k_]] = x_ < y_ ? x_ : y_;    \
        if ((t).kind[k_] != 1) (v)[(t).b[k_]] = x_ < y_ ? y_ : x_;    \
    }

}  // namespace net
}  // namespace gicp
