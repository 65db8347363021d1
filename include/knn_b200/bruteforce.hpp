// knn_b200/bruteforce.hpp -- C++ host API of the B200 engine, mirroring the
// reference's operator interface for the hot path (same names, argument
// meaning, ordering contract and exception text):
//
//   reference                                   here
//   knn::PointSet        point_set.hpp:14-49     knn_b200::PointSet
//   knn::Neighbor/Table  neighbor_table.hpp:11-44 knn_b200::Neighbor / NeighborTable
//   knn::Metric          metric.hpp:52-106       knn_b200::Metric
//   knn::BfConfig        bruteforce.hpp:12-20    knn_b200::BfConfig (+ engine path)
//   knn::SearchStats     bruteforce.hpp:22-25    knn_b200::SearchStats
//   knn::bf_knn          bruteforce.hpp:31-33    knn_b200::bf_knn
//   knn::bf_cost_model   bruteforce.hpp:35-43    knn_b200::bf_cost_model
//
// Header-only: every search goes through the C ABI (knn_b200.h) of
// libknn_b200.so.  Coordinates are narrowed to FP32 at the boundary (the
// engine's input type); reported distances are the engine's FP32 values
// widened to double.  Errors: std::invalid_argument with the reference's
// text for contract violations, std::runtime_error for device failures.
#pragma once

#include <cmath>
#include <cstddef>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../knn_b200.h"

namespace knn_b200 {

class PointSet {
public:
    PointSet(std::size_t n, std::size_t d, std::vector<double> data)
        : n_(n), d_(d), data_(std::move(data)) {
        // point_set.hpp:18-31, same order and text
        if (n_ == 0) throw std::invalid_argument("PointSet: point count must be >= 1");
        if (d_ == 0) throw std::invalid_argument("PointSet: dimension must be >= 1");
        if (data_.size() != n_ * d_)
            throw std::invalid_argument("PointSet: data size " + std::to_string(data_.size()) +
                                        " does not match " + std::to_string(n_) + "x" +
                                        std::to_string(d_));
        for (std::size_t i = 0; i < data_.size(); ++i)
            if (!std::isfinite(data_[i]))
                throw std::invalid_argument("PointSet: non-finite coordinate at point " +
                                            std::to_string(i / d_) + ", dimension " +
                                            std::to_string(i % d_));
    }
    std::size_t size() const { return n_; }
    std::size_t dim() const { return d_; }
    std::span<const double> row(std::size_t i) const { return {data_.data() + i * d_, d_}; }
    double coord(std::size_t i, std::size_t c) const { return data_[i * d_ + c]; }
    const std::vector<double>& data() const { return data_; }

    // FP32 copy handed to the engine.  The engine computes in FP32: a finite
    // coordinate beyond the FP32 range is rejected with its own message (it
    // would otherwise round to inf and read as "non-finite"); magnitudes below
    // the FP32 subnormal range round to +-0 (IEEE round-to-nearest).
    std::vector<float> as_f32(const char* which = "points") const {
        std::vector<float> out(data_.size());
        for (std::size_t i = 0; i < data_.size(); ++i) {
            out[i] = static_cast<float>(data_[i]);
            if (std::isinf(out[i]))
                throw std::invalid_argument(std::string("bf_knn: ") + which + " coordinate at point " +
                                            std::to_string(i / d_) + ", dimension " + std::to_string(i % d_) +
                                            " is outside the FP32 range of the engine (|x| > 3.4028235e38)");
        }
        return out;
    }

private:
    std::size_t n_, d_;
    std::vector<double> data_;
};

struct Neighbor {
    std::int64_t index;
    double distance;
    friend bool operator==(const Neighbor&, const Neighbor&) = default;
};

class NeighborTable {
public:
    NeighborTable(std::size_t query_count, std::size_t k)
        : n_(query_count), k_(k), entries_(query_count * k) {
        if (query_count == 0 || k == 0) throw std::invalid_argument("NeighborTable: empty table");
    }
    std::size_t query_count() const { return n_; }
    std::size_t k() const { return k_; }
    std::span<Neighbor> row(std::size_t i) { return {entries_.data() + i * k_, k_}; }
    std::span<const Neighbor> row(std::size_t i) const { return {entries_.data() + i * k_, k_}; }
    friend bool operator==(const NeighborTable& a, const NeighborTable& b) {
        return a.n_ == b.n_ && a.k_ == b.k_ && a.entries_ == b.entries_;
    }

private:
    std::size_t n_, k_;
    std::vector<Neighbor> entries_;
};

enum class MetricKind { euclidean = KNN_B200_EUCLIDEAN, manhattan = KNN_B200_MANHATTAN,
                        chebyshev = KNN_B200_CHEBYSHEV, mahalanobis = KNN_B200_MAHALANOBIS };

class Metric {
public:
    static Metric euclidean() { return Metric(MetricKind::euclidean); }
    static Metric manhattan() { return Metric(MetricKind::manhattan); }
    static Metric chebyshev() { return Metric(MetricKind::chebyshev); }

    // metric.cpp:20-61: validated at construction, same messages.
    static Metric mahalanobis(std::size_t d, std::vector<double> matrix) {
        if (d == 0) throw std::invalid_argument("Metric: Mahalanobis dimension must be >= 1");
        if (matrix.size() != d * d)
            throw std::invalid_argument("Metric: Mahalanobis matrix has " +
                                        std::to_string(matrix.size()) + " entries, expected " +
                                        std::to_string(d * d));
        for (std::size_t i = 0; i < d; ++i)
            for (std::size_t j = i + 1; j < d; ++j) {
                const double a = matrix[i * d + j], b = matrix[j * d + i];
                if (std::abs(a - b) > 1e-12 * std::max(std::abs(a), std::abs(b)))
                    throw std::invalid_argument("Metric: Mahalanobis matrix is not symmetric at (" +
                                                std::to_string(i) + "," + std::to_string(j) + ")");
            }
        std::vector<double> L(d * d, 0.0);  // Cholesky only to validate SPD
        for (std::size_t i = 0; i < d; ++i)
            for (std::size_t j = 0; j <= i; ++j) {
                double s = matrix[i * d + j];
                for (std::size_t c = 0; c < j; ++c) s -= L[i * d + c] * L[j * d + c];
                if (i == j) {
                    if (!(s > 0.0))
                        throw std::invalid_argument(
                            "Metric: Mahalanobis matrix is not positive definite (pivot " +
                            std::to_string(i) + ")");
                    L[i * d + i] = std::sqrt(s);
                } else {
                    L[i * d + j] = s / L[j * d + j];
                }
            }
        Metric m(MetricKind::mahalanobis);
        m.dim_ = d;
        m.matrix_ = std::move(matrix);
        return m;
    }

    MetricKind kind() const { return kind_; }
    std::size_t pinned_dim() const { return dim_; }
    const std::vector<double>& matrix() const { return matrix_; }

private:
    explicit Metric(MetricKind k) : kind_(k) {}
    MetricKind kind_;
    std::size_t dim_ = 0;
    std::vector<double> matrix_;
};

struct BfConfig {
    std::size_t chunk_size = 1024;       // accepted; never changes results
    unsigned worker_count = 0;           // accepted; never changes results
    bool count_distance_evals = false;
    int path = KNN_B200_PATH_AUTO;       // engine extension: exact / tensor / auto
    int device = -1;                     // engine extension: CUDA ordinal
};

struct SearchStats {
    std::uint64_t distance_evals = 0;
    std::uint64_t pruned_subtrees = 0;
};

// bruteforce.hpp:31-33: exhaustive exact kNN, rows ascending by distance, ties
// by ascending reference index, distances finalized (sqrt for the L2 kinds).
inline NeighborTable bf_knn(const PointSet& queries, const PointSet& references, std::size_t k,
                            const Metric& metric, const BfConfig& config = {},
                            SearchStats* stats = nullptr) {
    knn_b200_options o;
    knn_b200_options_init(&o);
    o.chunk_size = config.chunk_size;
    o.worker_count = config.worker_count;
    o.count_distance_evals = config.count_distance_evals ? 1 : 0;
    o.path = config.path;
    o.device = config.device;
    if (metric.kind() == MetricKind::mahalanobis) {
        o.mahalanobis = metric.matrix().data();
        o.mahalanobis_dim = static_cast<int64_t>(metric.pinned_dim());
    }
    const std::size_t n = queries.size();
    const std::vector<float> q = queries.as_f32("queries");
    const std::vector<float> r = references.as_f32("references");
    std::vector<float> dist(n * (k ? k : 1));
    std::vector<int64_t> idx(n * (k ? k : 1));
    uint64_t evals = 0;
    const knn_b200_status s = knn_b200_search(
        q.data(), static_cast<int64_t>(n), static_cast<int32_t>(queries.dim()), r.data(),
        static_cast<int64_t>(references.size()), static_cast<int32_t>(references.dim()),
        static_cast<int32_t>(k > 0x7fffffff ? 0x7fffffff : k), static_cast<int32_t>(metric.kind()),
        &o, dist.data(), idx.data(), &evals);
    if (s == KNN_B200_EINVAL) throw std::invalid_argument(knn_b200_last_error());
    if (s != KNN_B200_OK) throw std::runtime_error(knn_b200_last_error());
    NeighborTable table(n, k);
    for (std::size_t i = 0; i < n; ++i) {
        auto row = table.row(i);
        for (std::size_t t = 0; t < k; ++t)
            row[t] = {idx[i * k + t], static_cast<double>(dist[i * k + t])};
    }
    if (stats) stats->distance_evals = evals;  // bruteforce.cpp:98
    return table;
}

// bruteforce.hpp:35-43, bruteforce.cpp:102-112: the paper's closed-form
// operation counts of the exhaustive search.
struct BfCostModel {
    std::uint64_t additions;        // 2*n*m*d
    std::uint64_t multiplications;  // n*m*d
    double comparisons;             // n*m*log2(m)
};

inline BfCostModel bf_cost_model(std::size_t n, std::size_t m, std::size_t d, std::size_t k) {
    if (n == 0 || m == 0 || d == 0 || k == 0)
        throw std::invalid_argument("bf_cost_model: all inputs must be >= 1");
    const std::uint64_t nmd = static_cast<std::uint64_t>(n) * m * d;
    return BfCostModel{2 * nmd, nmd,
                       static_cast<double>(n) * static_cast<double>(m) *
                           std::log2(static_cast<double>(m))};
}

}  // namespace knn_b200
