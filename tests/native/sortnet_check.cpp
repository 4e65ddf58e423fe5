// Host check of the comparator networks of csrc/sortnet.cuh (tests/test_sortnet.py).
// Merge networks: every pair of sorted 0-1 runs (the 0-1 principle for merging), for
// all lengths used plus a sweep; sort networks: all 0-1 inputs up to N = 20 and
// random integer inputs (with ties) for larger N; pruned outputs checked likewise.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "../../paper_2308_07173_b200/csrc/sortnet.cuh"

using namespace gicp::net;

static void run(const Net& t, std::vector<unsigned>& v) {
    for (int k = 0; k < t.n; ++k) {
        const unsigned x = v[t.a[k]], y = v[t.b[k]];
        if (t.kind[k] != 2) v[t.a[k]] = std::min(x, y);
        if (t.kind[k] != 1) v[t.b[k]] = std::max(x, y);
    }
}

static int fails = 0;

template <int M, int B, int NOUT>
static void check_merge() {
    constexpr Net t = make_merge_net<M, B, NOUT>();
    std::mt19937 rng(M * 100 + B);
    for (int za = 0; za <= M; ++za)
        for (int zb = 0; zb <= B; ++zb) {
            std::vector<unsigned> v(M + B);
            for (int i = 0; i < M; ++i) v[i] = i < za ? 0 : 1;
            for (int i = 0; i < B; ++i) v[M + i] = i < zb ? 0 : 1;
            std::vector<unsigned> ref = v;
            std::sort(ref.begin(), ref.end());
            run(t, v);
            for (int r = 0; r < NOUT; ++r)
                if (v[t.out[r]] != ref[r]) {
                    ++fails;
                    std::printf("merge<%d,%d,%d> fails (za=%d zb=%d) at %d\n", M, B, NOUT, za, zb, r);
                    return;
                }
        }
    for (int it = 0; it < 20000; ++it) {
        std::vector<unsigned> a(M), b(B);
        for (auto& x : a) x = rng() % 50;
        for (auto& x : b) x = rng() % 50;
        std::sort(a.begin(), a.end());
        std::sort(b.begin(), b.end());
        std::vector<unsigned> v(a);
        v.insert(v.end(), b.begin(), b.end());
        std::vector<unsigned> ref = v;
        std::sort(ref.begin(), ref.end());
        run(t, v);
        for (int r = 0; r < NOUT; ++r)
            if (v[t.out[r]] != ref[r]) {
                ++fails;
                std::printf("merge<%d,%d,%d> random fails at %d\n", M, B, NOUT, r);
                return;
            }
    }
    std::printf("merge<%d,%d,%d>: %d ops ok\n", M, B, NOUT, t.n);
}

template <int N, int NOUT>
static void check_sort() {
    constexpr Net t = make_sort_net<N, NOUT>();
    if (N <= 20) {
        for (unsigned long long m = 0; m < (1ull << N); ++m) {
            std::vector<unsigned> v(N);
            for (int i = 0; i < N; ++i) v[i] = (m >> i) & 1;
            std::vector<unsigned> ref = v;
            std::sort(ref.begin(), ref.end());
            run(t, v);
            for (int r = 0; r < NOUT; ++r)
                if (v[t.out[r]] != ref[r]) {
                    ++fails;
                    std::printf("sort<%d,%d> fails on %llx\n", N, NOUT, m);
                    return;
                }
        }
    }
    std::mt19937 rng(N);
    for (int it = 0; it < 200000; ++it) {
        std::vector<unsigned> v(N);
        for (auto& x : v) x = rng() % (it & 1 ? 8 : 1000000);
        std::vector<unsigned> ref = v;
        std::sort(ref.begin(), ref.end());
        run(t, v);
        for (int r = 0; r < NOUT; ++r)
            if (v[t.out[r]] != ref[r]) {
                ++fails;
                std::printf("sort<%d,%d> random fails\n", N, NOUT);
                return;
            }
    }
    std::printf("sort<%d,%d>: %d ops ok\n", N, NOUT, t.n);
}

int main() {
    // the instantiations of knn_tile.cu (K + 1 list, 8-key buffer, 32-key first fill)
    check_merge<11, 8, 11>();
    check_merge<21, 8, 21>();
    check_merge<33, 8, 33>();
    check_sort<8, 8>();
    check_sort<16, 16>();
    check_sort<20, 20>();
    check_sort<32, 11>();
    check_sort<32, 21>();
    check_sort<32, 32>();
    // a sweep of merge shapes
    check_merge<1, 1, 2>();
    check_merge<1, 2, 3>();
    check_merge<2, 1, 3>();
    check_merge<3, 5, 8>();
    check_merge<5, 3, 6>();
    check_merge<7, 7, 14>();
    check_merge<13, 4, 10>();
    check_merge<17, 9, 26>();
    check_merge<20, 20, 40>();
    if (fails) {
        std::printf("FAILED %d\n", fails);
        return 1;
    }
    std::printf("ALL OK\n");
    return 0;
}
