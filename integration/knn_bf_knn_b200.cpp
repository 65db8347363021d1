// knn_bf_knn_b200.cpp -- the reference-side drop-in.
//
// A reference build (/root/reference/proj) links this translation unit
// INSTEAD OF src/bruteforce.cpp.  It defines the same two symbols with the
// same signatures, using the reference's own types from its headers:
//
//   knn::bf_knn          include/knn/bruteforce.hpp:31-33
//   knn::bf_cost_model   include/knn/bruteforce.hpp:35-43
//
// and forwards the search to the B200 engine through the C ABI
// (include/knn_b200.h).  Every caller of bf_knn -- knn-cli search, run_grid,
// rho_k / kl_entropy, knn_classify, retrieve_vote -- then
// runs on the GPU unchanged.  See INTEGRATION.md for the build recipe;
// oracle/Makefile's `dropin` target builds it with the reference's other
// sources plus integration/dropin_test.cpp.
#include <cmath>
#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "knn/bruteforce.hpp"
#include "knn_b200.h"

namespace knn {

// The engine computes in FP32 (north star).  A finite double beyond the FP32
// range would round to +-inf and then be reported by the engine as a
// "non-finite coordinate", which the reference never says for a finite input:
// reject it here with its own message.  Magnitudes below the FP32 subnormal
// range round to +-0 (IEEE round-to-nearest), which is the documented
// precision contract of the engine, not an error.
static std::vector<float> narrow_to_f32(const PointSet& p, const char* which) {
    const std::vector<double>& src = p.data();
    std::vector<float> out(src.size());
    for (std::size_t i = 0; i < src.size(); ++i) {
        out[i] = static_cast<float>(src[i]);
        if (std::isinf(out[i]))
            throw std::invalid_argument(std::string("bf_knn: ") + which + " coordinate at point " +
                                        std::to_string(i / p.dim()) + ", dimension " +
                                        std::to_string(i % p.dim()) +
                                        " is outside the FP32 range of the engine (|x| > 3.4028235e38)");
    }
    return out;
}

NeighborTable bf_knn(const PointSet& queries, const PointSet& references, std::size_t k,
                     const Metric& metric, const BfConfig& config, SearchStats* stats) {
    // The contract checks run here, before any whitening, so their order and
    // text are exactly bruteforce.cpp:44-56 (the engine repeats them).
    if (queries.dim() != references.dim())
        throw std::invalid_argument("bf_knn: dimension mismatch, queries have " +
                                    std::to_string(queries.dim()) + ", references have " +
                                    std::to_string(references.dim()));
    if (k == 0) throw std::invalid_argument("bf_knn: k must be >= 1");
    if (k > references.size())
        throw std::invalid_argument("bf_knn: k = " + std::to_string(k) +
                                    " exceeds reference count " +
                                    std::to_string(references.size()));
    if (config.chunk_size == 0) throw std::invalid_argument("bf_knn: chunk_size must be >= 1");
    metric.check_compatible(queries.dim());

    // Mahalanobis collapses to Euclidean on whitened points (metric.hpp:81-83);
    // whiten in double with the reference's own Metric::whiten.
    const PointSet* q = &queries;
    const PointSet* r = &references;
    std::optional<PointSet> wq, wr;
    if (metric.needs_whitening()) {
        wq.emplace(metric.whiten(queries));
        wr.emplace(metric.whiten(references));
        q = &*wq;
        r = &*wr;
    }
    int kind = KNN_B200_EUCLIDEAN;
    switch (metric.kernel_kind()) {
        case MetricKind::manhattan: kind = KNN_B200_MANHATTAN; break;
        case MetricKind::chebyshev: kind = KNN_B200_CHEBYSHEV; break;
        default: kind = KNN_B200_EUCLIDEAN; break;
    }

    const std::size_t n = q->size(), m = r->size(), d = q->dim();
    const std::vector<float> qf = narrow_to_f32(*q, "queries");
    const std::vector<float> rf = narrow_to_f32(*r, "references");
    std::vector<float> dist(n * k);
    std::vector<std::int64_t> idx(n * k);
    knn_b200_options o;
    knn_b200_options_init(&o);
    o.chunk_size = config.chunk_size;
    o.worker_count = config.worker_count;
    o.count_distance_evals = config.count_distance_evals ? 1 : 0;
    std::uint64_t evals = 0;
    const knn_b200_status s = knn_b200_search(
        qf.data(), static_cast<int64_t>(n), static_cast<int32_t>(d), rf.data(),
        static_cast<int64_t>(m), static_cast<int32_t>(d), static_cast<int32_t>(k), kind, &o,
        dist.data(), idx.data(), &evals);
    if (s == KNN_B200_EINVAL) throw std::invalid_argument(knn_b200_last_error());
    if (s != KNN_B200_OK) throw std::runtime_error(knn_b200_last_error());

    NeighborTable table(n, k);
    for (std::size_t i = 0; i < n; ++i) {
        auto row = table.row(i);
        for (std::size_t t = 0; t < k; ++t)
            row[t] = {idx[i * k + t], static_cast<double>(dist[i * k + t])};
    }
    if (stats) stats->distance_evals = evals;
    return table;
}

// The paper's operation counts, closed form.
BfCostModel bf_cost_model(std::size_t n, std::size_t m, std::size_t d, std::size_t k) {
    if (n == 0 || m == 0 || d == 0 || k == 0)
        throw std::invalid_argument("bf_cost_model: all inputs must be >= 1");
    const std::uint64_t nmd = static_cast<std::uint64_t>(n) * m * d;
    BfCostModel c{};
    c.additions = 2 * nmd;
    c.multiplications = nmd;
    c.comparisons = static_cast<double>(n) * static_cast<double>(m) * std::log2(static_cast<double>(m));
    return c;
}

}  // namespace knn
