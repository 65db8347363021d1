// test_bruteforce_b200.cpp -- the reference's hot-path unit tests
// (/root/reference/proj/tests/test_bruteforce.cpp), restated against the C++
// mirror API knn_b200::bf_knn.  Value checks use the north-star tolerance
// (1e-5 relative) instead of the reference's bitwise double equality, since
// the engine computes FP32 keys.
//
//   ./test_bruteforce_b200            all cases (needs a GPU)
//   ./test_bruteforce_b200 --no-gpu   host-side contract checks only
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <random>
#include <string>
#include <vector>

#include "knn_b200/bruteforce.hpp"

using knn_b200::BfConfig;
using knn_b200::Metric;
using knn_b200::NeighborTable;
using knn_b200::PointSet;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                                  \
    do {                                                                             \
        ++g_checks;                                                                  \
        if (!(cond)) {                                                               \
            ++g_fail;                                                                \
            std::printf("  CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond);   \
        }                                                                            \
    } while (0)

template <typename F>
static void check_throws(F&& f, const char* needle) {
    ++g_checks;
    try {
        f();
        ++g_fail;
        std::printf("  expected std::invalid_argument containing '%s'\n", needle);
    } catch (const std::invalid_argument& e) {
        if (!std::strstr(e.what(), needle)) {
            ++g_fail;
            std::printf("  message '%s' lacks '%s'\n", e.what(), needle);
        }
    }
}

static PointSet uniform_points(std::size_t n, std::size_t d, std::uint64_t seed, double lo = 0,
                               double hi = 1) {
    std::mt19937_64 gen(seed);
    std::vector<double> v(n * d);
    // FP32-exact values so the double oracle below sees the engine's inputs
    for (double& x : v) x = lo + (hi - lo) * static_cast<float>((gen() >> 40) * 0x1.0p-24);
    return PointSet(n, d, std::move(v));
}

// test_bruteforce.cpp:22-39
static void check_table_invariants(const NeighborTable& t, std::size_t m) {
    for (std::size_t i = 0; i < t.query_count(); ++i) {
        const auto row = t.row(i);
        std::vector<std::int64_t> seen;
        for (std::size_t j = 0; j < row.size(); ++j) {
            CHECK(row[j].index >= 0);
            CHECK(row[j].index < static_cast<std::int64_t>(m));
            seen.push_back(row[j].index);
            if (j > 0) {
                CHECK(row[j].distance >= row[j - 1].distance);
                if (row[j].distance == row[j - 1].distance) CHECK(row[j].index > row[j - 1].index);
            }
        }
        std::sort(seen.begin(), seen.end());
        CHECK(std::adjacent_find(seen.begin(), seen.end()) == seen.end());
    }
}

// serial double oracle (reference.cpp:11-51 semantics) + tolerance comparator
static void check_against_oracle(const PointSet& Q, const PointSet& R, std::size_t k,
                                 const NeighborTable& t, int metric) {
    for (std::size_t i = 0; i < Q.size(); ++i) {
        std::vector<std::pair<double, std::int64_t>> all;
        for (std::size_t j = 0; j < R.size(); ++j) {
            double acc = 0;
            for (std::size_t c = 0; c < Q.dim(); ++c) {
                const double df = Q.coord(i, c) - R.coord(j, c);
                if (metric == 0) acc += df * df;
                else if (metric == 1) acc += std::abs(df);
                else acc = std::max(acc, std::abs(df));
            }
            all.push_back({metric == 0 ? std::sqrt(acc) : acc, static_cast<std::int64_t>(j)});
        }
        std::sort(all.begin(), all.end());
        for (std::size_t r = 0; r < k; ++r) {
            const double ref = all[r].first, got = t.row(i)[r].distance;
            CHECK(std::abs(got - ref) <= 1e-5 * ref + 1e-6);
            if (t.row(i)[r].index != all[r].second) {
                // near-tie: the returned index's own distance must match rank r
                const std::int64_t j = t.row(i)[r].index;
                auto it = std::find_if(all.begin(), all.end(),
                                       [&](const auto& p) { return p.second == j; });
                CHECK(it != all.end() && std::abs(it->first - ref) <= 1e-5 * ref + 1e-6);
            }
        }
    }
}

static void contract_errors() {
    // test_bruteforce.cpp:92-102 (+ exact texts from bruteforce.cpp:44-56)
    const PointSet refs(3, 2, {0, 0, 1, 0, 2, 0});
    const PointSet query(1, 2, {0.1, 0});
    check_throws([&] { (void)knn_b200::bf_knn(query, refs, 4, Metric::euclidean()); },
                 "k = 4 exceeds reference count 3");
    check_throws([&] { (void)knn_b200::bf_knn(query, refs, 0, Metric::euclidean()); },
                 "k must be >= 1");
    const PointSet wrong_dim(1, 3, {0, 0, 0});
    check_throws([&] { (void)knn_b200::bf_knn(wrong_dim, refs, 1, Metric::euclidean()); },
                 "dimension mismatch, queries have 3, references have 2");
    BfConfig zero;
    zero.chunk_size = 0;
    check_throws([&] { (void)knn_b200::bf_knn(query, refs, 1, Metric::euclidean(), zero); },
                 "chunk_size must be >= 1");
    check_throws([&] { (void)PointSet(0, 2, {}); }, "point count must be >= 1");
    check_throws([&] { (void)PointSet(1, 2, {0, NAN}); }, "non-finite coordinate at point 0, dimension 1");
    check_throws([&] { (void)Metric::mahalanobis(2, {1, 2, 2, 1}); }, "not positive definite");
    // finite doubles beyond the FP32 range: the engine's own message, not "non-finite"
    const PointSet huge(1, 2, {0.5, 1e39});
    check_throws([&] { (void)knn_b200::bf_knn(huge, refs, 1, Metric::euclidean()); },
                 "queries coordinate at point 0, dimension 1 is outside the FP32 range");
    check_throws([&] { (void)knn_b200::bf_knn(query, PointSet(1, 2, {-4e38, 0}), 1, Metric::euclidean()); },
                 "references coordinate at point 0, dimension 0 is outside the FP32 range");
    check_throws(
        [&] {
            (void)knn_b200::bf_knn(query, refs, 1, Metric::mahalanobis(3, {1, 0, 0, 0, 1, 0, 0, 0, 1}));
        },
        "Mahalanobis matrix is 3x3 but points have dimension 2");
    // bf_cost_model (test_bruteforce.cpp cost cases; bruteforce.cpp:102-112)
    {
        const knn_b200::BfCostModel c = knn_b200::bf_cost_model(10, 100, 8, 5);
        CHECK(c.additions == 16000u);
        CHECK(c.multiplications == 8000u);
        CHECK(std::abs(c.comparisons - 1000.0 * std::log2(100.0)) < 1e-9);
        check_throws([&] { (void)knn_b200::bf_cost_model(0, 1, 1, 1); }, "all inputs must be >= 1");
    }
}

static void gpu_cases() {
    // collinear example and full sort (test_bruteforce.cpp:77-90)
    {
        const PointSet refs(3, 2, {0, 0, 1, 0, 2, 0});
        const PointSet query(1, 2, {0.1, 0});
        const NeighborTable t = knn_b200::bf_knn(query, refs, 2, Metric::euclidean());
        CHECK(t.row(0)[0].index == 0);
        CHECK(std::abs(t.row(0)[0].distance - 0.1) < 1e-6);
        CHECK(t.row(0)[1].index == 1);
        CHECK(std::abs(t.row(0)[1].distance - 0.9) < 1e-6);
        const NeighborTable full = knn_b200::bf_knn(query, refs, 3, Metric::euclidean());
        CHECK(full.row(0)[2].index == 2);
        check_table_invariants(full, 3);
    }
    // random instances vs the serial oracle, three metrics (test_bruteforce.cpp:104-122)
    {
        std::mt19937_64 gen(33);
        for (int trial = 0; trial < 12; ++trial) {
            const std::size_t n = 1 + gen() % 50, m = 1 + gen() % 50, k = 1 + gen() % m;
            const PointSet Q = uniform_points(n, 8, gen(), -2, 2);
            const PointSet R = uniform_points(m, 8, gen(), -2, 2);
            const int metric = trial % 3;
            const Metric mt = metric == 0 ? Metric::euclidean()
                              : metric == 1 ? Metric::manhattan()
                                            : Metric::chebyshev();
            const NeighborTable t = knn_b200::bf_knn(Q, R, k, mt);
            check_against_oracle(Q, R, k, t, metric);
            check_table_invariants(t, m);
        }
    }
    // determinism across workers / chunking and across engine paths
    // (test_bruteforce.cpp:124-136, acceptance C3)
    {
        const PointSet Q = uniform_points(37, 6, 101), R = uniform_points(53, 6, 102);
        const NeighborTable base = knn_b200::bf_knn(Q, R, 7, Metric::euclidean());
        for (unsigned w : {1u, 2u, 8u})
            for (std::size_t c : {std::size_t{1}, std::size_t{7}, Q.size()})
                for (int path : {KNN_B200_PATH_EXACT, KNN_B200_PATH_TENSOR, KNN_B200_PATH_AUTO}) {
                    BfConfig cfg;
                    cfg.worker_count = w;
                    cfg.chunk_size = c;
                    cfg.path = path;
                    CHECK(knn_b200::bf_knn(Q, R, 7, Metric::euclidean(), cfg) == base);
                }
    }
    // distance work does not depend on k (test_bruteforce.cpp:138-148)
    {
        const PointSet Q = uniform_points(30, 4, 55), R = uniform_points(40, 4, 56);
        BfConfig cfg;
        cfg.count_distance_evals = true;
        for (std::size_t k : {std::size_t{1}, std::size_t{20}, R.size()}) {
            knn_b200::SearchStats st;
            (void)knn_b200::bf_knn(Q, R, k, Metric::euclidean(), cfg, &st);
            CHECK(st.distance_evals == Q.size() * R.size());
        }
    }
    // all-duplicate data: ties resolve to the lowest indices (test_kdtree.cpp:65-75)
    {
        const PointSet P(64, 3, std::vector<double>(64 * 3, 1.5));
        const PointSet q(1, 3, {1.5, 1.5, 1.5});
        const NeighborTable t = knn_b200::bf_knn(q, P, 5, Metric::euclidean());
        for (std::size_t j = 0; j < 5; ++j) {
            CHECK(t.row(0)[j].index == static_cast<std::int64_t>(j));
            CHECK(t.row(0)[j].distance == 0.0);
        }
    }
    // Mahalanobis identity == Euclidean (test_core.cpp:40-51)
    {
        const PointSet p(1, 2, {1.0, 2.0}), q(1, 2, {4.0, 6.0});
        const NeighborTable t = knn_b200::bf_knn(p, q, 1, Metric::mahalanobis(2, {1, 0, 0, 1}));
        CHECK(std::abs(t.row(0)[0].distance - 5.0) < 1e-6);
    }
}

int main(int argc, char** argv) {
    const bool no_gpu = argc > 1 && std::strcmp(argv[1], "--no-gpu") == 0;
    std::printf("contract errors\n");
    contract_errors();
    if (!no_gpu) {
        std::printf("gpu cases\n");
        gpu_cases();
    }
    std::printf("%d checks, %d failed\n", g_checks, g_fail);
    return g_fail == 0 ? 0 : 1;
}
