// ref_capi.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" wrapper compiled TOGETHER WITH the unmodified reference
// sources (/root/reference/proj/src/{bruteforce,topk,metric,reference,
// entropy,applications}.cpp) into oracle/_ref/libknnref.so by oracle/Makefile.
// It lets the Python test-suite and bench.py's reference arm call the
// reference's own knn::bf_knn / knn::reference_knn through ctypes.  Nothing in
// the product package links this library.
//
// Entry points wrapped (paths relative to /root/reference/proj):
//   knn::bf_knn          include/knn/bruteforce.hpp:31-33
//   knn::reference_knn   include/knn/reference.hpp:15-16
//   knn::rho_k_all       include/knn/entropy.hpp (self-join caller of bf_knn)
//   knn::knn_classify / knn::retrieve_vote   include/knn/applications.hpp
//   knn::derive_seed / next_unit   include/knn/rng.hpp:17-38
#include <cstdint>
#include <cstring>
#include <exception>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include <omp.h>

#include "knn/applications.hpp"
#include "knn/bruteforce.hpp"
#include "knn/entropy.hpp"
#include "knn/metric.hpp"
#include "knn/reference.hpp"
#include "knn/rng.hpp"

namespace {

knn::Metric make_metric(int kind, std::size_t d, const double* mahal) {
    switch (kind) {
        case 1: return knn::Metric::manhattan();
        case 2: return knn::Metric::chebyshev();
        case 3: return knn::Metric::mahalanobis(d, std::vector<double>(mahal, mahal + d * d));
        default: return knn::Metric::euclidean();
    }
}

void copy_err(const std::exception& e, char* err, std::size_t errlen) {
    if (err && errlen) {
        std::strncpy(err, e.what(), errlen - 1);
        err[errlen - 1] = '\0';
    }
}

void unpack(const knn::NeighborTable& t, std::int64_t* idx, double* dist) {
    for (std::size_t i = 0; i < t.query_count(); ++i) {
        auto row = t.row(i);
        for (std::size_t j = 0; j < t.k(); ++j) {
            idx[i * t.k() + j] = row[j].index;
            dist[i * t.k() + j] = row[j].distance;
        }
    }
}

}  // namespace

extern "C" {

// Returns 0 on success, 1 for std::invalid_argument, 2 for any other exception;
// the exception text is copied into err.
int knnref_bf_knn(const double* Q, std::size_t n, const double* R, std::size_t m,
                  std::size_t dq, std::size_t dr, std::size_t k, int metric,
                  const double* mahal, std::size_t mahal_d, std::size_t chunk,
                  unsigned workers, int count_evals, std::int64_t* out_idx,
                  double* out_dist, std::uint64_t* evals, char* err, std::size_t errlen) {
    try {
        knn::PointSet q(n, dq, std::vector<double>(Q, Q + n * dq));
        knn::PointSet r(m, dr, std::vector<double>(R, R + m * dr));
        knn::BfConfig cfg;
        cfg.chunk_size = chunk;
        cfg.worker_count = workers;
        cfg.count_distance_evals = count_evals != 0;
        knn::SearchStats stats;
        knn::NeighborTable t =
            knn::bf_knn(q, r, k, make_metric(metric, mahal_d, mahal), cfg, &stats);
        unpack(t, out_idx, out_dist);
        if (evals) *evals = stats.distance_evals;
        return 0;
    } catch (const std::invalid_argument& e) {
        copy_err(e, err, errlen);
        return 1;
    } catch (const std::exception& e) {
        copy_err(e, err, errlen);
        return 2;
    }
}

int knnref_reference_knn(const double* Q, std::size_t n, const double* R, std::size_t m,
                         std::size_t d, std::size_t k, int metric, const double* mahal,
                         std::int64_t* out_idx, double* out_dist, char* err,
                         std::size_t errlen) {
    try {
        knn::PointSet q(n, d, std::vector<double>(Q, Q + n * d));
        knn::PointSet r(m, d, std::vector<double>(R, R + m * d));
        unpack(knn::reference_knn(q, r, k, make_metric(metric, d, mahal)), out_idx, out_dist);
        return 0;
    } catch (const std::invalid_argument& e) {
        copy_err(e, err, errlen);
        return 1;
    } catch (const std::exception& e) {
        copy_err(e, err, errlen);
        return 2;
    }
}

int knnref_rho_k_all(const double* P, std::size_t n, std::size_t d, std::size_t k,
                     double* out, char* err, std::size_t errlen) {
    try {
        knn::PointSet p(n, d, std::vector<double>(P, P + n * d));
        std::vector<double> rho = knn::rho_k_all(p, k);
        std::memcpy(out, rho.data(), n * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        copy_err(e, err, errlen);
        return 1;
    }
}

int knnref_knn_classify(const double* T, std::size_t m, std::size_t dt, const std::int64_t* labels,
                        std::size_t nlabels, const double* Q, std::size_t n, std::size_t dq,
                        std::size_t k, int metric, std::int64_t* out, char* err,
                        std::size_t errlen) {
    try {
        knn::LabeledSet train(knn::PointSet(m, dt, std::vector<double>(T, T + m * dt)),
                              std::vector<std::int64_t>(labels, labels + nlabels));
        knn::PointSet q(n, dq, std::vector<double>(Q, Q + n * dq));
        const auto r = knn::knn_classify(train, q, k, make_metric(metric, dq, nullptr));
        std::memcpy(out, r.data(), n * sizeof(std::int64_t));
        return 0;
    } catch (const std::invalid_argument& e) {
        copy_err(e, err, errlen);
        return 1;
    } catch (const std::exception& e) {
        copy_err(e, err, errlen);
        return 2;
    }
}

int knnref_retrieve_vote(const double* D, std::size_t m, std::size_t dd, const std::int64_t* owners,
                         std::size_t nowners, std::int64_t images, const double* Q, std::size_t n,
                         std::size_t dq, std::size_t k, int metric, std::uint64_t* scores,
                         std::int64_t* ranking, char* err, std::size_t errlen) {
    try {
        knn::DescriptorDatabase db(knn::PointSet(m, dd, std::vector<double>(D, D + m * dd)),
                                   std::vector<std::int64_t>(owners, owners + nowners), images);
        knn::PointSet q(n, dq, std::vector<double>(Q, Q + n * dq));
        const knn::VoteTally t = knn::retrieve_vote(db, q, k, make_metric(metric, dq, nullptr));
        std::memcpy(scores, t.scores.data(), t.scores.size() * sizeof(std::uint64_t));
        std::memcpy(ranking, t.ranking.data(), t.ranking.size() * sizeof(std::int64_t));
        return 0;
    } catch (const std::invalid_argument& e) {
        copy_err(e, err, errlen);
        return 1;
    } catch (const std::exception& e) {
        copy_err(e, err, errlen);
        return 2;
    }
}

std::uint64_t knnref_derive_seed(std::uint64_t master, std::uint64_t a, std::uint64_t b,
                                 std::uint64_t c) {
    return knn::derive_seed(master, a, b, c);
}

// generate_uniform's draw sequence (bench.cpp:39-46) without pulling in the
// JSON-dependent bench.cpp: mt19937_64 through knn::next_unit.
void knnref_uniform(std::uint64_t seed, double* out, std::size_t count) {
    std::mt19937_64 gen(seed);
    for (std::size_t i = 0; i < count; ++i) out[i] = knn::next_unit(gen);
}

void knnref_mt64_draws(std::uint64_t seed, std::uint64_t* out, std::size_t count) {
    std::mt19937_64 gen(seed);
    for (std::size_t i = 0; i < count; ++i) out[i] = gen();
}

int knnref_max_threads(void) { return omp_get_max_threads(); }

}  // extern "C"
