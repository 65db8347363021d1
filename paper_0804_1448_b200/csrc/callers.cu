// callers.cu -- the hot path's next consumers on the device (SURVEY.md 8(f)
// rank 3): the self-join behind the entropy estimator and the two voting
// applications.  Each is one engine search followed by a small epilogue
// kernel over the n x k table in HBM, so only the final answers come back.
//
//   rho_k_all      entropy.cpp:48-57,75-89: bf_knn(points, points, k + 1),
//                  then per point the k-th neighbour distance with the point
//                  itself excluded BY INDEX (a coincident point with another
//                  index still counts, at distance 0).
//   knn_classify   applications.cpp:36-63: majority vote over the k labels;
//                  ties by the smaller summed distance (summed in rank order,
//                  in double, like the reference's std::map tally), then by the
//                  smaller label token.
//   retrieve_vote  applications.cpp:65-86: every neighbour votes for its
//                  owning image (integer counts: exact), ranking by descending
//                  score, ties by ascending image id.
//
// Symmetry of the self-join (Q == R) is not exploited: the filter's epilogue
// scans rows (thread = query) of an A = ||r||^2 - 2 q.r tile, and the
// transposed view of the same tile is a different matrix (||q||^2 - 2 q.r)
// that would need column-wise group minima across lanes -- more epilogue work
// than the halved MMA saves while the epilogue, not the tensor pipe, binds.
#include <algorithm>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/knn_b200.h"
#include "common.cuh"
#include "engine.cuh"
#include "profile.cuh"

namespace knnb200 {
namespace {

// one thread per point: the k-th entry of its (k+1)-list after skipping self
__global__ void extract_rho_kernel(const float* dist, const int64_t* idx, int64_t n, int kp1,
                                   double* out) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float* dr = dist + i * kp1;
    const int64_t* ir = idx + i * kp1;
    int kept = 0;
    double rho = 0.0;
    for (int t = 0; t < kp1; ++t) {
        if (ir[t] == i) continue;
        rho = static_cast<double>(dr[t]);
        if (++kept == kp1 - 1) break;
    }
    out[i] = rho;
}

// one warp per query: for every rank j (lane-strided) the votes and the
// rank-ordered distance sum of its label; the best (votes desc, sum asc,
// label asc) by a warp reduction
__global__ void classify_kernel(const float* dist, const int64_t* idx, const int64_t* labels,
                                int64_t n, int k, int64_t* out) {
    const int64_t q = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (q >= n) return;
    const float* dr = dist + q * k;
    const int64_t* ir = idx + q * k;
    int best_v = -1;
    double best_s = 0.0;
    int64_t best_l = 0;
    for (int j = lane; j < k; j += 32) {
        const int64_t lj = __ldg(labels + ir[j]);
        int v = 0;
        double s = 0.0;
        for (int t = 0; t < k; ++t) {  // rank order, like the reference's tally
            if (__ldg(labels + ir[t]) == lj) {
                ++v;
                s += static_cast<double>(dr[t]);
            }
        }
        if (v > best_v || (v == best_v && (s < best_s || (s == best_s && lj < best_l)))) {
            best_v = v;
            best_s = s;
            best_l = lj;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const int v = __shfl_xor_sync(0xffffffffu, best_v, o);
        const double s = __shfl_xor_sync(0xffffffffu, best_s, o);
        const int64_t l = __shfl_xor_sync(0xffffffffu, best_l, o);
        if (v > best_v || (v == best_v && (s < best_s || (s == best_s && l < best_l)))) {
            best_v = v;
            best_s = s;
            best_l = l;
        }
    }
    if (lane == 0) out[q] = best_l;
}

// one thread per (query, rank): a vote for the owning image
__global__ void vote_kernel(const int64_t* idx, int64_t total, const int64_t* image_of,
                            unsigned long long* scores) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= total) return;
    atomicAdd(scores + __ldg(image_of + idx[t]), 1ull);
}

unsigned blocks(int64_t threads, int per = 256) {
    return static_cast<unsigned>((threads + per - 1) / per);
}

template <typename T>
struct DevBuf {  // stream-ordered scratch of one call
    T* p = nullptr;
    cudaStream_t s;
    DevBuf(size_t count, cudaStream_t st) : s(st) {
        KNN_CUDA_CHECK(cudaMallocAsync(&p, sizeof(T) * std::max<size_t>(count, 1), s));
    }
    ~DevBuf() {
        if (p) cudaFreeAsync(p, s);
    }
};

template <typename F>
knn_b200_status guarded(F&& body) {
    return static_cast<knn_b200_status>(abi_guarded(std::forward<F>(body)));
}

void rethrow(knn_b200_status st) {
    if (st == KNN_B200_OK) return;
    const std::string msg = knn_b200_last_error();
    switch (st) {
        case KNN_B200_EINVAL: throw InvalidArgument(msg);
        case KNN_B200_ENOMEM: throw OutOfMemory(msg);
        case KNN_B200_ECUDA: throw CudaError(msg);
        default: throw std::runtime_error(msg);
    }
}

// engine stream of the device selected by the options (synchronous calls)
cudaStream_t engine_stream(const knn_b200_options& o) {
    DeviceContext& ctx = context_for(o.device);
    KNN_CUDA_CHECK(cudaSetDevice(ctx.device));
    return ctx.stream;
}

void rho_device(const float* d_points, int64_t n, int d, int k, const knn_b200_options& o,
                cudaStream_t s, double* d_out) {
    if (k <= 0 || k >= n)
        throw InvalidArgument("rho_k_all: k = " + std::to_string(k) +
                              " needs at least k + 1 points, set has " + std::to_string(n));
    DevBuf<float> dd(static_cast<size_t>(n) * (k + 1), s);
    DevBuf<int64_t> di(static_cast<size_t>(n) * (k + 1), s);
    knn_b200_options so = o;  // a synchronous caller (no stream) searches on the engine
    so.raw_keys = 0;          // stream s, synchronized and value-checked like PointSet
    rethrow(knn_b200_search_device(d_points, n, d_points, n, d, k + 1, KNN_B200_EUCLIDEAN, &so,
                                   dd.p, di.p));
    {
        ProfileScope ps(s, "rho_extract_kernel");
        extract_rho_kernel<<<blocks(n), 256, 0, s>>>(dd.p, di.p, n, k + 1, d_out);
    }
    KNN_LAUNCH_CHECK();
}

}  // namespace
}  // namespace knnb200

using namespace knnb200;

extern "C" {

knn_b200_status knn_b200_rho_k_all_device(const float* d_points, int64_t n, int32_t d, int32_t k,
                                          const knn_b200_options* opt, double* d_out_rho) {
    return guarded([&] {
        knn_b200_options o;
        if (opt) o = *opt;
        else knn_b200_options_init(&o);
        if (!d_points || !d_out_rho) throw InvalidArgument("rho_k_all: null pointer");
        const bool sync = !o.stream;
        cudaStream_t s = sync ? engine_stream(o) : static_cast<cudaStream_t>(o.stream);
        rho_device(d_points, n, d, k, o, s, d_out_rho);
        if (sync) KNN_CUDA_CHECK(cudaStreamSynchronize(s));
    });
}

knn_b200_status knn_b200_rho_k_all(const float* points, int64_t n, int32_t d, int32_t k,
                                   const knn_b200_options* opt, double* out_rho) {
    return guarded([&] {
        knn_b200_options o;
        if (opt) o = *opt;
        else knn_b200_options_init(&o);
        if (!points || !out_rho) throw InvalidArgument("rho_k_all: null pointer");
        if (n <= 0) throw InvalidArgument("PointSet: point count must be >= 1");
        if (d <= 0) throw InvalidArgument("PointSet: dimension must be >= 1");
        cudaStream_t s = engine_stream(o);
        DevBuf<float> dp(static_cast<size_t>(n) * d, s);
        DevBuf<double> dr(static_cast<size_t>(n), s);
        KNN_CUDA_CHECK(cudaMemcpyAsync(dp.p, points, sizeof(float) * n * d, cudaMemcpyHostToDevice, s));
        knn_b200_options so = o;
        so.stream = nullptr;  // synchronous inner search: values validated like PointSet
        rho_device(dp.p, n, d, k, so, s, dr.p);
        KNN_CUDA_CHECK(cudaMemcpyAsync(out_rho, dr.p, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
        KNN_CUDA_CHECK(cudaStreamSynchronize(s));
    });
}

knn_b200_status knn_b200_knn_classify(const float* train, int64_t m, int32_t d,
                                      const int64_t* labels, const float* queries, int64_t n,
                                      int32_t dq, int32_t k, int32_t metric,
                                      const knn_b200_options* opt, int64_t* out_labels) {
    return guarded([&] {
        knn_b200_options o;
        if (opt) o = *opt;
        else knn_b200_options_init(&o);
        if (!train || !labels || !queries || !out_labels)
            throw InvalidArgument("knn_classify: null pointer");
        if (m <= 0 || n <= 0) throw InvalidArgument("PointSet: point count must be >= 1");
        if (d <= 0 || dq <= 0) throw InvalidArgument("PointSet: dimension must be >= 1");
        cudaStream_t s = engine_stream(o);
        DevBuf<float> dt(static_cast<size_t>(m) * d, s);
        DevBuf<float> dqv(static_cast<size_t>(n) * dq, s);
        DevBuf<int64_t> dl(static_cast<size_t>(m), s);
        DevBuf<float> dd(static_cast<size_t>(n) * std::max(k, 1), s);
        DevBuf<int64_t> di(static_cast<size_t>(n) * std::max(k, 1), s);
        DevBuf<int64_t> dout(static_cast<size_t>(n), s);
        KNN_CUDA_CHECK(cudaMemcpyAsync(dt.p, train, sizeof(float) * m * d, cudaMemcpyHostToDevice, s));
        KNN_CUDA_CHECK(cudaMemcpyAsync(dqv.p, queries, sizeof(float) * n * dq, cudaMemcpyHostToDevice, s));
        KNN_CUDA_CHECK(cudaMemcpyAsync(dl.p, labels, sizeof(int64_t) * m, cudaMemcpyHostToDevice, s));
        // the reference's order: PointSet values (construction), then bf_knn
        check_finite_device(s, dt.p, m, d, nullptr);
        check_finite_device(s, dqv.p, n, dq, nullptr);
        if (dq != d)
            throw InvalidArgument("bf_knn: dimension mismatch, queries have " + std::to_string(dq) +
                                  ", references have " + std::to_string(d));
        knn_b200_options so = o;
        so.stream = nullptr;
        rethrow(knn_b200_search_device(dqv.p, n, dt.p, m, d, k, metric, &so, dd.p, di.p));
        {
            ProfileScope ps(s, "classify_vote_kernel");
            classify_kernel<<<blocks(n * 32), 256, 0, s>>>(dd.p, di.p, dl.p, n, k, dout.p);
        }
        KNN_LAUNCH_CHECK();
        KNN_CUDA_CHECK(cudaMemcpyAsync(out_labels, dout.p, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, s));
        KNN_CUDA_CHECK(cudaStreamSynchronize(s));
    });
}

knn_b200_status knn_b200_retrieve_vote(const float* descriptors, int64_t m, int32_t d,
                                       const int64_t* image_of, int64_t image_count,
                                       const float* queries, int64_t n, int32_t dq, int32_t k,
                                       int32_t metric, const knn_b200_options* opt,
                                       uint64_t* out_scores, int64_t* out_ranking) {
    return guarded([&] {
        knn_b200_options o;
        if (opt) o = *opt;
        else knn_b200_options_init(&o);
        if (!descriptors || !image_of || !queries || !out_scores || !out_ranking)
            throw InvalidArgument("retrieve_vote: null pointer");
        if (m <= 0 || n <= 0) throw InvalidArgument("PointSet: point count must be >= 1");
        if (d <= 0 || dq <= 0) throw InvalidArgument("PointSet: dimension must be >= 1");
        // DescriptorDatabase (applications.cpp:9-34), in its order
        if (image_count <= 0) throw InvalidArgument("DescriptorDatabase: image count must be >= 1");
        std::vector<char> seen(static_cast<size_t>(image_count), 0);
        for (int64_t i = 0; i < m; ++i) {
            const int64_t id = image_of[i];
            if (id < 0 || id >= image_count)
                throw InvalidArgument("DescriptorDatabase: image identifier " + std::to_string(id) +
                                      " outside [0, " + std::to_string(image_count) + ")");
            seen[static_cast<size_t>(id)] = 1;
        }
        for (int64_t id = 0; id < image_count; ++id)
            if (!seen[static_cast<size_t>(id)])
                throw InvalidArgument("DescriptorDatabase: image " + std::to_string(id) +
                                      " owns no descriptors");
        if (dq != d)
            throw InvalidArgument("bf_knn: dimension mismatch, queries have " + std::to_string(dq) +
                                  ", references have " + std::to_string(d));
        cudaStream_t s = engine_stream(o);
        DevBuf<float> dt(static_cast<size_t>(m) * d, s);
        DevBuf<float> dqv(static_cast<size_t>(n) * d, s);
        DevBuf<int64_t> downer(static_cast<size_t>(m), s);
        DevBuf<float> dd(static_cast<size_t>(n) * std::max(k, 1), s);
        DevBuf<int64_t> di(static_cast<size_t>(n) * std::max(k, 1), s);
        DevBuf<unsigned long long> dsc(static_cast<size_t>(image_count), s);
        KNN_CUDA_CHECK(cudaMemcpyAsync(dt.p, descriptors, sizeof(float) * m * d, cudaMemcpyHostToDevice, s));
        KNN_CUDA_CHECK(cudaMemcpyAsync(dqv.p, queries, sizeof(float) * n * d, cudaMemcpyHostToDevice, s));
        KNN_CUDA_CHECK(cudaMemcpyAsync(downer.p, image_of, sizeof(int64_t) * m, cudaMemcpyHostToDevice, s));
        KNN_CUDA_CHECK(cudaMemsetAsync(dsc.p, 0, sizeof(unsigned long long) * image_count, s));
        check_finite_device(s, dt.p, m, d, nullptr);
        check_finite_device(s, dqv.p, n, d, nullptr);
        knn_b200_options so = o;
        so.stream = nullptr;
        rethrow(knn_b200_search_device(dqv.p, n, dt.p, m, d, k, metric, &so, dd.p, di.p));
        {
            ProfileScope ps(s, "retrieve_vote_kernel");
            vote_kernel<<<blocks(n * k), 256, 0, s>>>(di.p, n * k, downer.p, dsc.p);
        }
        KNN_LAUNCH_CHECK();
        KNN_CUDA_CHECK(cudaMemcpyAsync(out_scores, dsc.p, sizeof(uint64_t) * image_count,
                                       cudaMemcpyDeviceToHost, s));
        KNN_CUDA_CHECK(cudaStreamSynchronize(s));
        // ranking: descending score, ties by ascending identifier (applications.cpp:78-84)
        std::iota(out_ranking, out_ranking + image_count, int64_t{0});
        std::sort(out_ranking, out_ranking + image_count, [&](int64_t a, int64_t b) {
            return out_scores[a] > out_scores[b] || (out_scores[a] == out_scores[b] && a < b);
        });
    });
}

}  // extern "C"
