// dropin_test.cpp -- the reference's own callers of bf_knn, running on the B200
// engine through integration/knn_bf_knn_b200.cpp (linked in place of the
// reference's src/bruteforce.cpp).  Built by oracle/Makefile `dropin` from the
// unmodified reference sources; run by tests/test_dropin_gpu.py.
//
// Checks (reference anchors relative to /root/reference/proj):
//   C1  bf_knn vs the serial oracle reference_knn, 4 metrics   acceptance.cpp:58-84
//   KAT rho_k on {0,1,3} and duplicates                        test_entropy.cpp:60-72
//   C4  kl_entropy of a Gaussian sample within 0.05 nats       acceptance.cpp:131-139
//   C10 knn_classify k=1 == label of the nearest neighbour     acceptance.cpp:248-264
//       retrieve_vote ranks the generating image first, votes sum to n*k
//   C9  distance_evals == n*m for any k                        acceptance.cpp:225-235
// Distances are compared with the north-star tolerance (1e-5 relative) and
// indices allowed to differ only at near-ties, since the engine's keys are FP32.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <numbers>
#include <random>
#include <string>
#include <vector>

#include "knn/applications.hpp"
#include "knn/bruteforce.hpp"
#include "knn/entropy.hpp"
#include "knn/metric.hpp"
#include "knn/reference.hpp"
#include "knn/rng.hpp"

using namespace knn;

static int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                              \
    do {                                                                      \
        ++g_checks;                                                           \
        if (!(c)) {                                                           \
            ++g_fail;                                                         \
            std::printf("  CHECK failed line %d: %s\n", __LINE__, #c);        \
        }                                                                     \
    } while (0)

static PointSet fp32_uniform(std::size_t n, std::size_t d, std::uint64_t seed, double lo, double hi) {
    std::mt19937_64 gen(seed);
    std::vector<double> v(n * d);
    for (double& x : v) x = static_cast<float>(lo + (hi - lo) * next_unit(gen));
    return PointSet(n, d, std::move(v));
}

static PointSet fp32_gaussian(std::size_t n, std::size_t d, std::uint64_t seed) {
    std::mt19937_64 gen(seed);
    std::vector<double> v(n * d);
    for (double& x : v) {
        const double u1 = (static_cast<double>(gen() >> 11) + 0.5) * 0x1.0p-53;
        const double u2 = next_unit(gen);
        x = static_cast<float>(std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * std::numbers::pi * u2));
    }
    return PointSet(n, d, std::move(v));
}

static void compare_tables(const NeighborTable& got, const NeighborTable& ref, const PointSet& Q,
                           const PointSet& R, const Metric& metric) {
    for (std::size_t i = 0; i < ref.query_count(); ++i)
        for (std::size_t t = 0; t < ref.k(); ++t) {
            const double d_ref = ref.row(i)[t].distance, d_got = got.row(i)[t].distance;
            CHECK(std::abs(d_got - d_ref) <= 1e-5 * d_ref + 1e-6);
            if (got.row(i)[t].index != ref.row(i)[t].index) {
                const double dj = distance(Q.row(i), R.row(static_cast<std::size_t>(got.row(i)[t].index)), metric);
                CHECK(std::abs(dj - d_ref) <= 1e-5 * d_ref + 1e-6);
            }
        }
}

int main() {
    // C1: random instances, four metrics, vs the serial full-sort oracle
    {
        std::mt19937_64 gen(1001);
        const std::vector<double> spd{2.0, 0.4, 0.0, 0.4, 1.5, -0.2, 0.0, -0.2, 1.0};
        for (int trial = 0; trial < 40; ++trial) {
            const std::size_t n = 1 + gen() % 200, m = 1 + gen() % 200;
            const std::size_t d = trial % 4 == 3 ? 3 : 1 + gen() % 32;
            const std::size_t k = 1 + gen() % m;
            const Metric metric = trial % 4 == 0   ? Metric::euclidean()
                                  : trial % 4 == 1 ? Metric::manhattan()
                                  : trial % 4 == 2 ? Metric::chebyshev()
                                                   : Metric::mahalanobis(3, spd);
            const PointSet Q = fp32_uniform(n, d, gen(), -5, 5), R = fp32_uniform(m, d, gen(), -5, 5);
            compare_tables(bf_knn(Q, R, k, metric), reference_knn(Q, R, k, metric), Q, R, metric);
        }
    }
    // rho_k known answers (self-join through bf_knn(points, points, k+1))
    {
        const PointSet line(3, 1, {0, 1, 3});
        CHECK(rho_k(line, 0, 1) == 1.0);
        CHECK(rho_k(line, 0, 2) == 3.0);
        CHECK(rho_k(line, 2, 1) == 2.0);
        const PointSet dup(3, 1, {5, 5, 9});
        CHECK(rho_k(dup, 0, 1) == 0.0);
        CHECK(rho_k(dup, 2, 1) == 4.0);
    }
    // C4: Kozachenko-Leonenko entropy of a 1-d Gaussian (10000-point self-join)
    {
        EntropyConfig cfg;
        cfg.k = 5;
        const double est = kl_entropy(fp32_gaussian(10000, 1, 42), cfg).value_nats;
        const double truth = 0.5 * std::log(2.0 * std::numbers::pi * std::numbers::e);
        std::printf("  kl_entropy %.4f vs %.4f\n", est, truth);
        CHECK(std::abs(est - truth) < 0.05);
    }
    // C10: classification and retrieval on top of bf_knn
    {
        std::mt19937_64 gen(7007);
        for (int trial = 0; trial < 20; ++trial) {
            const std::size_t m = 2 + gen() % 80;
            const PointSet pts = fp32_uniform(m, 2 + gen() % 4, gen(), 0, 1);
            std::vector<std::int64_t> labels(m);
            for (auto& l : labels) l = static_cast<std::int64_t>(gen() % 6);
            const LabeledSet train(pts, labels);
            const PointSet queries = fp32_uniform(5, pts.dim(), gen(), 0, 1);
            const auto pred = knn_classify(train, queries, 1, Metric::euclidean());
            const auto table = bf_knn(queries, pts, 1, Metric::euclidean());
            for (std::size_t i = 0; i < queries.size(); ++i)
                CHECK(pred[i] == labels[static_cast<std::size_t>(table.row(i)[0].index)]);
        }
        // 5 images x 20 descriptors far apart, queries drawn from image 3
        std::vector<double> data, qd;
        std::vector<std::int64_t> owners;
        std::mt19937_64 g2(42);
        for (int img = 0; img < 5; ++img)
            for (int p = 0; p < 20; ++p) {
                owners.push_back(img);
                for (int c = 0; c < 4; ++c) data.push_back(static_cast<float>(50.0 * img + next_unit(g2)));
            }
        for (int i = 0; i < 10; ++i)
            for (int c = 0; c < 4; ++c) qd.push_back(static_cast<float>(150.0 + next_unit(g2)));
        const DescriptorDatabase db(PointSet(100, 4, data), owners, 5);
        const VoteTally tally = retrieve_vote(db, PointSet(10, 4, qd), 5, Metric::euclidean());
        CHECK(tally.ranking[0] == 3);
        std::uint64_t sum = 0;
        for (auto s : tally.scores) sum += s;
        CHECK(sum == 10 * 5);
    }
    // C9: evaluation count is exactly n*m for any k
    {
        const PointSet R = fp32_uniform(500, 6, 6006, 0, 1), Q = fp32_uniform(100, 6, 6007, 0, 1);
        BfConfig cfg;
        cfg.count_distance_evals = true;
        for (std::size_t k : {std::size_t{1}, std::size_t{20}, R.size()}) {
            SearchStats st;
            (void)bf_knn(Q, R, k, Metric::euclidean(), cfg, &st);
            CHECK(st.distance_evals == Q.size() * R.size());
        }
        const auto c = bf_cost_model(10, 100, 8, 5);
        CHECK(c.multiplications == 8000 && c.additions == 16000);
    }
    std::printf("%d checks, %d failed\n", g_checks, g_fail);
    return g_fail == 0 ? 0 : 1;
}
