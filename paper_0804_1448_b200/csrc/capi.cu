// capi.cu -- the extern "C" boundary (include/knn_b200.h).
//
// Validation order and exception text follow the reference exactly
// (paths relative to /root/reference/proj):
//   PointSet construction ........ include/knn/point_set.hpp:18-31
//   Metric::mahalanobis .......... src/metric.cpp:20-61
//   bf_knn ....................... src/bruteforce.cpp:44-56
//   Metric::check_compatible ..... include/knn/metric.hpp:90-96
// Invalid arguments map to KNN_B200_EINVAL with that text in
// knn_b200_last_error(); the C++ mirror rethrows them as std::invalid_argument.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "../../include/knn_b200.h"
#include "common.cuh"
#include "engine.cuh"
#include "exact_kernel.cuh"
#include "tensor_path.cuh"

namespace knnb200 {

namespace {
thread_local std::string g_last_error;
thread_local uint64_t g_launches = 0;

template <typename F>
knn_b200_status guarded(F&& body) {
    return static_cast<knn_b200_status>(abi_guarded(std::forward<F>(body)));
}

const knn_b200_options& opts_or_default(const knn_b200_options* opt, knn_b200_options& tmp) {
    if (opt) return *opt;
    knn_b200_options_init(&tmp);
    return tmp;
}

void check_point_set(const float* data, int64_t n, int64_t d, bool check_values) {
    if (n <= 0) throw InvalidArgument("PointSet: point count must be >= 1");
    if (d <= 0) throw InvalidArgument("PointSet: dimension must be >= 1");
    if (!data) throw InvalidArgument("PointSet: null data pointer");
    if (!check_values) return;
    const int64_t total = n * d;
    for (int64_t i = 0; i < total; ++i) {
        if (!std::isfinite(data[i])) {
            throw InvalidArgument("PointSet: non-finite coordinate at point " +
                                  std::to_string(i / d) + ", dimension " +
                                  std::to_string(i % d));
        }
    }
}

// Device-side PointSet value check (point_set.hpp:27-31): first index of a
// non-finite coordinate (atomicMin), so the host API validates a device copy
// in microseconds instead of scanning n*d values on one host core.
unsigned scan_grid(int64_t count);

// 16-byte loads over the aligned middle, four in flight per thread.
__global__ void finite_scan_kernel(const float* X, int64_t count, unsigned long long* first,
                                   int64_t base = 0) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const int64_t h = std::min<int64_t>(count, ((16 - (reinterpret_cast<uintptr_t>(X) & 15)) & 15) / 4);
    const int64_t n4 = (count - h) / 4;
    const float4* X4 = reinterpret_cast<const float4*>(X + h);
    auto bad = [&](int64_t i) { atomicMin(first, static_cast<unsigned long long>(base + i)); };
    for (int64_t i = t; i < h; i += stride)
        if (!isfinite(__ldg(X + i))) bad(i);
    for (int64_t i0 = t; i0 < n4; i0 += 4 * stride) {
        float4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
            v[u] = i0 + u * stride < n4 ? __ldg(X4 + i0 + u * stride) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const float c[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (!isfinite(c[j])) {
                    bad(h + 4 * (i0 + u * stride) + j);
                    break;
                }
        }
    }
    for (int64_t i = h + 4 * n4 + t; i < count; i += stride)
        if (!isfinite(__ldg(X + i))) bad(i);
}

// No CUDA device (e.g. a CPU-only CI box): validate on the host so argument
// errors keep the reference's text; the search itself then fails loudly.
bool device_present() {
    static const bool present = [] {
        int count = 0;
        return cudaGetDeviceCount(&count) == cudaSuccess && count > 0;
    }();
    return present;
}

void throw_non_finite(unsigned long long i, int64_t d) {
    throw InvalidArgument("PointSet: non-finite coordinate at point " +
                          std::to_string(static_cast<int64_t>(i) / d) + ", dimension " +
                          std::to_string(static_cast<int64_t>(i) % d));
}

}  // namespace

// Device-input value check (point_set.hpp:27-31) for the synchronous device
// APIs: first non-finite coordinate, with the reference's message.
void check_finite_device(cudaStream_t s, const float* X, int64_t rows, int64_t d,
                         unsigned long long* dbad) {
    // persistent per-device result slot (device) and pinned host copy: no
    // allocation per call (a stream-ordered malloc/free pair re-maps pool
    // memory after every synchronisation -- hundreds of microseconds)
    struct Slots {
        unsigned long long* dev = nullptr;
        unsigned long long* host = nullptr;
    };
    static std::mutex mu;
    static std::map<int, Slots> per_device;
    int device = 0;
    KNN_CUDA_CHECK(cudaGetDevice(&device));
    std::lock_guard<std::mutex> lock(mu);  // one check at a time per process (slot reuse)
    Slots& sl = per_device[device];
    if (!sl.dev) {
        KNN_CUDA_CHECK(cudaMalloc(&sl.dev, sizeof(unsigned long long)));
        KNN_CUDA_CHECK(cudaMallocHost(&sl.host, sizeof(unsigned long long)));
    }
    unsigned long long* tmp = dbad ? dbad : sl.dev;
    const int64_t count = rows * d;
    KNN_CUDA_CHECK(cudaMemsetAsync(tmp, 0xff, sizeof(unsigned long long), s));
    finite_scan_kernel<<<scan_grid(count), 256, 0, s>>>(X, count, tmp);
    KNN_LAUNCH_CHECK();
    KNN_CUDA_CHECK(cudaMemcpyAsync(sl.host, tmp, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    KNN_CUDA_CHECK(cudaStreamSynchronize(s));
    const unsigned long long bad = *sl.host;
    if (bad != ~0ull) throw_non_finite(bad, d);
}

namespace {

// Metric::mahalanobis (metric.cpp:20-61): validate, Cholesky M = L L^T.
std::vector<double> cholesky_or_throw(const double* M, int64_t d) {
    if (d <= 0) throw InvalidArgument("Metric: Mahalanobis dimension must be >= 1");
    if (!M) throw InvalidArgument("Metric: Mahalanobis matrix has 0 entries, expected " +
                                  std::to_string(d * d));
    for (int64_t i = 0; i < d; ++i)
        for (int64_t j = i + 1; j < d; ++j) {
            const double a = M[i * d + j], b = M[j * d + i];
            if (std::abs(a - b) > 1e-12 * std::max(std::abs(a), std::abs(b)))
                throw InvalidArgument("Metric: Mahalanobis matrix is not symmetric at (" +
                                      std::to_string(i) + "," + std::to_string(j) + ")");
        }
    std::vector<double> L(static_cast<size_t>(d * d), 0.0);
    for (int64_t i = 0; i < d; ++i)
        for (int64_t j = 0; j <= i; ++j) {
            double s = M[i * d + j];
            for (int64_t c = 0; c < j; ++c) s -= L[i * d + c] * L[j * d + c];
            if (i == j) {
                if (!(s > 0.0))
                    throw InvalidArgument(
                        "Metric: Mahalanobis matrix is not positive definite (pivot " +
                        std::to_string(i) + ")");
                L[i * d + i] = std::sqrt(s);
            } else {
                L[i * d + j] = s / L[j * d + j];
            }
        }
    return L;
}

// y = L^T x in double on widened inputs (metric.cpp:63-82), narrowed to FP32
// for the Euclidean kernel the metric collapses to (metric.hpp:81-83).
std::vector<float> whiten(const std::vector<double>& L, const float* x, int64_t n, int64_t d) {
    std::vector<float> out(static_cast<size_t>(n * d));
    std::vector<double> row(static_cast<size_t>(d));
    for (int64_t p = 0; p < n; ++p) {
        for (int64_t c = 0; c < d; ++c) row[c] = x[p * d + c];
        for (int64_t r = 0; r < d; ++r) {
            double acc = 0.0;
            for (int64_t c = r; c < d; ++c) acc += L[c * d + r] * row[c];
            out[p * d + r] = static_cast<float>(acc);
        }
    }
    return out;
}

// Device whitening, bitwise equal to whiten(): y_r = sum_{c >= r} L[c][r] x_c
// with round-to-nearest double multiplies and adds in ascending c, narrowed to
// FP32.  In place: a block stages each point's row (as double) in shared
// memory before overwriting it.  LT = L^T row-major (LT[r][c] = L[c][r]).
constexpr int kWhitenMaxD = 8192;  // row staging: d doubles of shared memory

__global__ void __launch_bounds__(128) whiten_kernel(float* X, int64_t n, int d, const double* LT) {
    extern __shared__ double xs[];
    for (int64_t p = blockIdx.x; p < n; p += gridDim.x) {
        float* row = X + p * d;
        for (int c = threadIdx.x; c < d; c += blockDim.x) xs[c] = static_cast<double>(row[c]);
        __syncthreads();
        for (int r = threadIdx.x; r < d; r += blockDim.x) {
            const double* lt = LT + static_cast<int64_t>(r) * d;
            double acc = 0.0;
            for (int c = r; c < d; ++c) acc = __dadd_rn(acc, __dmul_rn(__ldg(lt + c), xs[c]));
            row[r] = __double2float_rn(acc);
        }
        __syncthreads();
    }
}

// Whiten device rows in place (Q and R of one search) with the Cholesky factor
// L (host, d x d row-major); dLT: device scratch of d*d doubles.
void whiten_device(cudaStream_t s, const std::vector<double>& L, int d, double* dLT, float* X1,
                   int64_t n1, float* X2, int64_t n2) {
    std::vector<double> LT(static_cast<size_t>(d) * d);
    for (int r = 0; r < d; ++r)
        for (int c = 0; c < d; ++c) LT[static_cast<size_t>(r) * d + c] = L[static_cast<size_t>(c) * d + r];
    KNN_CUDA_CHECK(cudaMemcpyAsync(dLT, LT.data(), sizeof(double) * LT.size(), cudaMemcpyHostToDevice, s));
    const size_t smem = sizeof(double) * d;
    if (smem > 48 * 1024)
        KNN_CUDA_CHECK(cudaFuncSetAttribute(whiten_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            static_cast<int>(smem)));
    for (auto [X, n] : {std::pair<float*, int64_t>{X1, n1}, std::pair<float*, int64_t>{X2, n2}}) {
        if (n == 0) continue;
        const unsigned grid = static_cast<unsigned>(std::min<int64_t>(n, 148 * 16));
        whiten_kernel<<<grid, 128, smem, s>>>(X, n, d, dLT);
        KNN_LAUNCH_CHECK();
    }
    // the host copy of LT must outlive the async copy
    KNN_CUDA_CHECK(cudaStreamSynchronize(s));
}

// bruteforce.cpp:44-56 in order, then Metric::check_compatible.
void check_search(int64_t dq, int64_t dr, int64_t m, int64_t k, const knn_b200_options& o,
                  int metric) {
    if (dq != dr)
        throw InvalidArgument("bf_knn: dimension mismatch, queries have " + std::to_string(dq) +
                              ", references have " + std::to_string(dr));
    if (k <= 0) throw InvalidArgument("bf_knn: k must be >= 1");
    if (k > m)
        throw InvalidArgument("bf_knn: k = " + std::to_string(k) + " exceeds reference count " +
                              std::to_string(m));
    if (o.chunk_size == 0) throw InvalidArgument("bf_knn: chunk_size must be >= 1");
    if (metric < 0 || metric > 3) throw InvalidArgument("bf_knn: unknown metric");
    if (metric == kMahalanobis && o.mahalanobis_dim != dq)
        throw InvalidArgument("Metric: Mahalanobis matrix is " + std::to_string(o.mahalanobis_dim) +
                              "x" + std::to_string(o.mahalanobis_dim) +
                              " but points have dimension " + std::to_string(dq));
    if (k > 0x7ffffffe || m > 0x7ffffffe)
        throw InvalidArgument("bf_knn: k and m must be < 2^31 per device search");
}

}  // namespace

void note_launch(int count) { g_launches += static_cast<uint64_t>(count); }

void set_last_error(const std::string& msg) { g_last_error = msg; }

}  // namespace knnb200

using namespace knnb200;

struct knn_b200_index {
    int device = 0;
    const float* dR = nullptr;
    bool owned = false;
    int64_t m = 0;
    int d = 0;
    int64_t base = 0;
    std::mutex mu;
    // tensor path: the reference set prepared once, when the index is created
    // (fp16 copy, norms, radii), reused by every search on any stream (the
    // KdTree build/search split, kdtree.hpp:21,70-72)
    knnb200::TensorRefs tref;
    void* tref_mem = nullptr;
    ~knn_b200_index() {
        if (owned && dR) cudaFree(const_cast<float*>(dR));
        if (tref_mem) cudaFree(tref_mem);
    }
};

namespace knnb200 {
namespace {
const TensorRefs* index_refs(knn_b200_index* h, int64_t n, int k, int metric, int path) {
    if (plan_search(n, h->m, h->d, k, metric, path).path != 2 || !h->tref_mem) return nullptr;
    return &h->tref;
}

// Eager tensor-path preparation of an index's reference set (d <= 128), on
// the engine stream and synchronized: searches on any stream may use it.
void prepare_index(DeviceContext& ctx, knn_b200_index* h) {
    if (!tensor_path_supported(1, h->m, h->d, 1)) return;
    KNN_CUDA_CHECK(cudaMalloc(&h->tref_mem, tensor_refs_bytes(h->m, h->d)));
    tensor_prep_refs(ctx.stream, h->dR, h->m, h->d, h->tref_mem, h->tref);
    KNN_CUDA_CHECK(cudaStreamSynchronize(ctx.stream));
}
}  // namespace
}  // namespace knnb200

namespace knnb200 {
namespace {

// queries per pipeline stage (multiple of 256): large enough that a chunk's
// search runs near full efficiency (one chunk per ~128 query-tile pairs)
// largest query chunk of the pipelined host search (dev knob KNN_B200_PIPE_CHUNK);
// below 2 x half of it, one staged search
int64_t pipe_chunk() {
    static const int64_t v = [] {
        const char* e = getenv("KNN_B200_PIPE_CHUNK");
        return e ? std::max<int64_t>(512, atoll(e)) : int64_t{32768};
    }();
    return v;
}

unsigned scan_grid(int64_t count) {
    return static_cast<unsigned>(std::min<int64_t>((count + 255) / 256, 1184));
}

// One-shot host search, staged: H2D of both sets, device value check, search, D2H.
void search_staged(DeviceContext& ctx, const float* q, int64_t n, const float* r, int64_t m,
                   int dq, int dr, int k, int metric, int path, int raw_keys, bool host_values,
                   float* out_dist, int64_t* out_idx, const std::vector<double>* chol = nullptr) {
    cudaStream_t s = ctx.stream;
    Sizer sz;
    sz.take<float>(static_cast<size_t>(n) * dq);
    sz.take<float>(static_cast<size_t>(m) * dr);
    sz.take<float>(static_cast<size_t>(n) * k);
    sz.take<int64_t>(static_cast<size_t>(n) * k);
    sz.take<unsigned long long>(2);
    if (chol) sz.take<double>(static_cast<size_t>(dq) * dq);
    ctx.s->io.reserve(sz.used + 256);
    Carver cv{static_cast<char*>(ctx.s->io.base())};
    float* dQ = cv.take<float>(static_cast<size_t>(n) * dq);
    float* dR = cv.take<float>(static_cast<size_t>(m) * dr);
    float* dO = cv.take<float>(static_cast<size_t>(n) * k);
    int64_t* dI = cv.take<int64_t>(static_cast<size_t>(n) * k);
    unsigned long long* dbad = cv.take<unsigned long long>(2);
    KNN_CUDA_CHECK(cudaMemcpyAsync(dQ, q, sizeof(float) * n * dq, cudaMemcpyHostToDevice, s));
    KNN_CUDA_CHECK(cudaMemcpyAsync(dR, r, sizeof(float) * m * dr, cudaMemcpyHostToDevice, s));
    if (chol) {  // Mahalanobis: whiten on the device, then the Euclidean kernel
        double* dLT = cv.take<double>(static_cast<size_t>(dq) * dq);
        whiten_device(s, *chol, dq, dLT, dQ, n, dR, m);
    }
    if (!host_values) {
        KNN_CUDA_CHECK(cudaMemsetAsync(dbad, 0xff, 2 * sizeof(unsigned long long), s));
        finite_scan_kernel<<<scan_grid(n * dq), 256, 0, s>>>(dQ, n * dq, dbad);
        KNN_LAUNCH_CHECK();
        finite_scan_kernel<<<scan_grid(m * dr), 256, 0, s>>>(dR, m * dr, dbad + 1);
        KNN_LAUNCH_CHECK();
        unsigned long long bad[2];
        KNN_CUDA_CHECK(cudaMemcpyAsync(bad, dbad, sizeof(bad), cudaMemcpyDeviceToHost, s));
        KNN_CUDA_CHECK(cudaStreamSynchronize(s));
        if (bad[0] != ~0ull) throw_non_finite(bad[0], dq);
        if (bad[1] != ~0ull) throw_non_finite(bad[1], dr);
    }
    search_device(ctx, s, dQ, n, dR, m, dq, k, metric, path, raw_keys, 0, dO, dI);
    KNN_CUDA_CHECK(cudaMemcpyAsync(out_dist, dO, sizeof(float) * n * k, cudaMemcpyDeviceToHost, s));
    KNN_CUDA_CHECK(cudaMemcpyAsync(out_idx, dI, sizeof(int64_t) * n * k, cudaMemcpyDeviceToHost, s));
    KNN_CUDA_CHECK(cudaStreamSynchronize(s));
}

// One-shot host search on the tensor path, pipelined over query chunks: the
// reference set is copied and prepared once, then chunk c's H2D (copy stream)
// overlaps chunk c-1's search (compute stream), whose D2H overlaps chunk c's
// search.  Coordinates are validated on the device and checked before any
// result is returned; certification fallbacks of all chunks are collected and
// resolved once at the end.
// Query chunk boundaries of the pipelined host search: equal chunks of at
// most pipe_chunk() queries, at least two, multiples of the 256-query tile
// pair.  Dev knob KNN_B200_PIPE_CHUNKS="a,b,c": explicit leading chunk sizes
// (rounded to 256), the rest in one chunk.
static std::vector<int64_t> pipe_schedule(int64_t n) {
    std::vector<int64_t> st{0};
    if (const char* e = std::getenv("KNN_B200_PIPE_CHUNKS")) {
        const char* p = e;
        while (*p && st.back() < n) {
            char* end = nullptr;
            const long long v = std::strtoll(p, &end, 10);
            if (end == p) break;
            const int64_t sz = std::max<int64_t>(256, (v + 255) / 256 * 256);
            st.push_back(std::min(n, st.back() + sz));
            p = *end == ',' ? end + 1 : end;
        }
        if (st.back() < n) st.push_back(n);
        return st;
    }
    const int64_t chunks = std::max<int64_t>(2, (n + pipe_chunk() - 1) / pipe_chunk());
    const int64_t csz = ((n + chunks - 1) / chunks + 255) / 256 * 256;
    for (int64_t q0 = csz; q0 < n; q0 += csz) st.push_back(q0);
    st.push_back(n);
    return st;
}

void search_pipelined(DeviceContext& ctx, const float* q, int64_t n, const float* r, int64_t m,
                      int d, int k, int raw_keys, float* out_dist, int64_t* out_idx) {
    cudaStream_t s = ctx.stream, cs = ctx.copy_stream;
    Sizer sz;
    sz.take<float>(static_cast<size_t>(n) * d);
    sz.take<float>(static_cast<size_t>(m) * d);
    sz.take<float>(static_cast<size_t>(n) * k);
    sz.take<int64_t>(static_cast<size_t>(n) * k);
    sz.take<unsigned long long>(2);
    sz.take<int>(static_cast<size_t>(n) + 1);
    const size_t fb_part = fallback_part_elems(n, m, k);
    const size_t fb_glist = fallback_glist_elems(k);
    sz.take<float>(fb_part);
    sz.take<int64_t>(fb_part);
    sz.take<float>(fb_glist);
    sz.take<int32_t>(fb_glist);
    ctx.s->io.reserve(sz.used + 256);
    ctx.s->refs.reserve(tensor_refs_bytes(m, d));
    Carver cv{static_cast<char*>(ctx.s->io.base())};
    float* dQ = cv.take<float>(static_cast<size_t>(n) * d);
    float* dR = cv.take<float>(static_cast<size_t>(m) * d);
    float* dO = cv.take<float>(static_cast<size_t>(n) * k);
    int64_t* dI = cv.take<int64_t>(static_cast<size_t>(n) * k);
    unsigned long long* dbad = cv.take<unsigned long long>(2);
    int* fb = cv.take<int>(static_cast<size_t>(n) + 1);
    float* fb_pk = cv.take<float>(fb_part);
    int64_t* fb_pi = cv.take<int64_t>(fb_part);
    float* fb_gk = cv.take<float>(fb_glist);
    int32_t* fb_gi = cv.take<int32_t>(fb_glist);
    KNN_CUDA_CHECK(cudaMemsetAsync(dbad, 0xff, 2 * sizeof(unsigned long long), s));
    KNN_CUDA_CHECK(cudaMemsetAsync(fb, 0, sizeof(int), s));
    // every H2D goes through the copy stream in order (R, then the query
    // chunks): the reference prep overlaps the first chunk's copy
    KNN_CUDA_CHECK(cudaEventRecord(ctx.ev[0], s));
    KNN_CUDA_CHECK(cudaStreamWaitEvent(cs, ctx.ev[0], 0));
    KNN_CUDA_CHECK(cudaMemcpyAsync(dR, r, sizeof(float) * m * d, cudaMemcpyHostToDevice, cs));
    KNN_CUDA_CHECK(cudaEventRecord(ctx.ev[15], cs));
    KNN_CUDA_CHECK(cudaStreamWaitEvent(s, ctx.ev[15], 0));
    finite_scan_kernel<<<scan_grid(m * d), 256, 0, s>>>(dR, m * d, dbad + 1);
    KNN_LAUNCH_CHECK();
    TensorRefs refs;
    tensor_prep_refs(s, dR, m, d, ctx.s->refs.base(), refs);
    // chunks of <= pipe_chunk() queries, at least two (n >= pipe_chunk() here),
    // multiples of the 256-query tile pair
    std::vector<int64_t> cstart = pipe_schedule(n);
    FallbackSink sink{fb, fb + 1, 0};
    const int64_t nch = static_cast<int64_t>(cstart.size()) - 1;
    while (static_cast<int64_t>(ctx.pipe_ev.size()) < 2 * nch) {
        cudaEvent_t e;
        KNN_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        ctx.pipe_ev.push_back(e);
    }
    // 1. every chunk's H2D, back to back on the copy stream (a chunk's D2H
    //    queued between them would hold the next copy behind a search)
    for (int64_t c = 0; c < nch; ++c) {
        const int64_t q0 = cstart[c], nq = cstart[c + 1] - q0;
        KNN_CUDA_CHECK(cudaMemcpyAsync(dQ + q0 * d, q + q0 * d, sizeof(float) * nq * d,
                                       cudaMemcpyHostToDevice, cs));
        KNN_CUDA_CHECK(cudaEventRecord(ctx.pipe_ev[2 * c], cs));
    }
    // 2. per chunk: validate + search as soon as its rows landed; its D2H
    //    (copy stream, after all H2D) overlaps the next chunk's search
    for (int64_t c = 0; c < nch; ++c) {
        const int64_t q0 = cstart[c], nq = cstart[c + 1] - q0;
        KNN_CUDA_CHECK(cudaStreamWaitEvent(s, ctx.pipe_ev[2 * c], 0));
        finite_scan_kernel<<<scan_grid(nq * d), 256, 0, s>>>(dQ + q0 * d, nq * d, dbad, q0 * d);
        KNN_LAUNCH_CHECK();
        sink.offset = static_cast<int>(q0);
        tensor_search(ctx, s, refs, dQ + q0 * d, nq, k, raw_keys, 0, dO + q0 * k, dI + q0 * k,
                      &sink);
        KNN_CUDA_CHECK(cudaEventRecord(ctx.pipe_ev[2 * c + 1], s));
        KNN_CUDA_CHECK(cudaStreamWaitEvent(cs, ctx.pipe_ev[2 * c + 1], 0));
        KNN_CUDA_CHECK(cudaMemcpyAsync(out_dist + q0 * k, dO + q0 * k, sizeof(float) * nq * k,
                                       cudaMemcpyDeviceToHost, cs));
        KNN_CUDA_CHECK(cudaMemcpyAsync(out_idx + q0 * k, dI + q0 * k, sizeof(int64_t) * nq * k,
                                       cudaMemcpyDeviceToHost, cs));
    }
    // uncertified queries of all chunks, resolved once over the whole query
    // set (small k on the device: exact kernel over the recorded list)
    tensor_resolve_fallbacks(ctx, s, refs, dQ, n, k, raw_keys, 0, dO, dI, fb, fb_pk, fb_pi, fb_gk, fb_gi);
    unsigned long long bad[2];
    int fails = 0;
    KNN_CUDA_CHECK(cudaMemcpyAsync(bad, dbad, sizeof(bad), cudaMemcpyDeviceToHost, s));
    KNN_CUDA_CHECK(cudaMemcpyAsync(&fails, fb, sizeof(int), cudaMemcpyDeviceToHost, s));
    KNN_CUDA_CHECK(cudaStreamSynchronize(s));
    KNN_CUDA_CHECK(cudaStreamSynchronize(cs));
    if (bad[0] != ~0ull) throw_non_finite(bad[0], d);
    if (bad[1] != ~0ull) throw_non_finite(bad[1], d);
    if (!ctx.s->fb_on_device) fails = ctx.s->last_fallbacks;
    ctx.s->last_fallbacks = fails;
    ctx.s->fb_on_device = false;
    if (fails == 0) return;
    // the chunk results already copied back predate the fallback: copy again
    KNN_CUDA_CHECK(cudaMemcpyAsync(out_dist, dO, sizeof(float) * n * k, cudaMemcpyDeviceToHost, s));
    KNN_CUDA_CHECK(cudaMemcpyAsync(out_idx, dI, sizeof(int64_t) * n * k, cudaMemcpyDeviceToHost, s));
    KNN_CUDA_CHECK(cudaStreamSynchronize(s));
}

}  // namespace
}  // namespace knnb200

extern "C" {

void knn_b200_options_init(knn_b200_options* opt) {
    if (!opt) return;
    std::memset(opt, 0, sizeof(*opt));
    opt->struct_size = sizeof(*opt);
    opt->device = -1;
    opt->path = KNN_B200_PATH_AUTO;
    opt->chunk_size = 1024;  // BfConfig default (bruteforce.hpp:15)
}

const char* knn_b200_last_error(void) { return g_last_error.c_str(); }

const char* knn_b200_version(void) { return "knn_b200 0.1 (sm_100a)"; }

uint64_t knn_b200_launch_count(void) { return g_launches; }
void knn_b200_reset_launch_count(void) { g_launches = 0; }

knn_b200_status knn_b200_search(const float* queries, int64_t n, int32_t dq,
                                const float* references, int64_t m, int32_t dr, int32_t k,
                                int32_t metric, const knn_b200_options* opt, float* out_dist,
                                int64_t* out_idx, uint64_t* distance_evals) {
    return guarded([&] {
        knn_b200_options tmp;
        const knn_b200_options& o = opts_or_default(opt, tmp);
        std::vector<double> chol;
        if (metric == kMahalanobis) chol = cholesky_or_throw(o.mahalanobis, o.mahalanobis_dim);
        // values are checked on the device below (Euclidean / L1 / Linf); the
        // host scan only runs where the reference's error order needs it
        const bool host_values = metric == kMahalanobis || !device_present();
        check_point_set(queries, n, dq, host_values);
        check_point_set(references, m, dr, host_values);
        try {
            check_search(dq, dr, m, k, o, metric);
        } catch (const InvalidArgument&) {
            // a PointSet error is raised at construction, before any bf_knn check
            check_point_set(queries, n, dq, true);
            check_point_set(references, m, dr, true);
            throw;
        }
        if (!out_dist || !out_idx) throw InvalidArgument("bf_knn: null output pointer");

        std::vector<float> wq, wr;
        const float* q = queries;
        const float* r = references;
        int kernel_metric = metric;
        bool device_whiten = false;
        if (metric == kMahalanobis) {
            kernel_metric = kL2;
            device_whiten = device_present() && dq <= kWhitenMaxD;
            if (!device_whiten) {  // the reference's own host step (metric.cpp:63-82)
                wq = whiten(chol, queries, n, dq);
                wr = whiten(chol, references, m, dr);
                q = wq.data();
                r = wr.data();
            }
        }

        DeviceContext& ctx = context_for(o.device);
        std::lock_guard<std::mutex> lock(ctx.mu);
        KNN_CUDA_CHECK(cudaSetDevice(ctx.device));
        ctx.bind(ctx.stream);
        if (plan_search(n, m, dq, k, kernel_metric, o.path).path == 2 && !host_values &&
            n >= pipe_chunk())
            search_pipelined(ctx, q, n, r, m, dq, k, o.raw_keys, out_dist, out_idx);
        else
            search_staged(ctx, q, n, r, m, dq, dr, k, kernel_metric, o.path, o.raw_keys, host_values,
                          out_dist, out_idx, device_whiten ? &chol : nullptr);
        if (distance_evals)
            *distance_evals = o.count_distance_evals ? static_cast<uint64_t>(n) * m : 0;
    });
}

knn_b200_status knn_b200_search_device(const float* d_queries, int64_t n,
                                       const float* d_references, int64_t m, int32_t d,
                                       int32_t k, int32_t metric, const knn_b200_options* opt,
                                       float* d_out_dist, int64_t* d_out_idx) {
    return guarded([&] {
        knn_b200_options tmp;
        const knn_b200_options& o = opts_or_default(opt, tmp);
        std::vector<double> chol;
        if (metric == kMahalanobis) chol = cholesky_or_throw(o.mahalanobis, o.mahalanobis_dim);
        check_point_set(d_queries, n, d, false);
        check_point_set(d_references, m, d, false);
        check_search(d, d, m, k, o, metric);
        if (!d_out_dist || !d_out_idx) throw InvalidArgument("bf_knn: null output pointer");
        if (metric == kMahalanobis && d > kWhitenMaxD)
            throw InvalidArgument("knn_b200_search_device: Mahalanobis needs d <= " +
                                  std::to_string(kWhitenMaxD));
        DeviceContext& ctx = context_for(o.device);
        std::lock_guard<std::mutex> lock(ctx.mu);
        KNN_CUDA_CHECK(cudaSetDevice(ctx.device));
        cudaStream_t s = o.stream ? static_cast<cudaStream_t>(o.stream) : ctx.stream;
        ctx.bind(s);
        if (!o.stream) {  // synchronous call: validate the values like PointSet does
            check_finite_device(s, d_queries, n, d, nullptr);
            check_finite_device(s, d_references, m, d, nullptr);
        }
        const float* q = d_queries;
        const float* r = d_references;
        int kernel_metric = metric;
        if (metric == kMahalanobis) {  // whitened copies (the inputs are the caller's)
            Sizer sz;
            sz.take<float>(static_cast<size_t>(n) * d);
            sz.take<float>(static_cast<size_t>(m) * d);
            sz.take<double>(static_cast<size_t>(d) * d);
            ctx.s->io.reserve(sz.used + 256);
            Carver cv{static_cast<char*>(ctx.s->io.base())};
            float* wq = cv.take<float>(static_cast<size_t>(n) * d);
            float* wr = cv.take<float>(static_cast<size_t>(m) * d);
            double* dLT = cv.take<double>(static_cast<size_t>(d) * d);
            KNN_CUDA_CHECK(cudaMemcpyAsync(wq, q, sizeof(float) * n * d, cudaMemcpyDeviceToDevice, s));
            KNN_CUDA_CHECK(cudaMemcpyAsync(wr, r, sizeof(float) * m * d, cudaMemcpyDeviceToDevice, s));
            whiten_device(s, chol, d, dLT, wq, n, wr, m);
            q = wq;
            r = wr;
            kernel_metric = kL2;
        }
        search_device(ctx, s, q, n, r, m, d, k, kernel_metric, o.path, o.raw_keys, 0, d_out_dist,
                      d_out_idx);
        if (!o.stream) KNN_CUDA_CHECK(cudaStreamSynchronize(s));
    });
}

knn_b200_status knn_b200_index_create(const float* references, int64_t m, int32_t d,
                                      int64_t index_base, const knn_b200_options* opt,
                                      knn_b200_index** out) {
    return guarded([&] {
        knn_b200_options tmp;
        const knn_b200_options& o = opts_or_default(opt, tmp);
        if (!out) throw InvalidArgument("knn_b200_index_create: null out");
        check_point_set(references, m, d, true);
        DeviceContext& ctx = context_for(o.device);
        KNN_CUDA_CHECK(cudaSetDevice(ctx.device));
        auto* h = new knn_b200_index();
        h->device = ctx.device;
        h->m = m;
        h->d = d;
        h->base = index_base;
        float* p = nullptr;
        cudaError_t e = cudaMalloc(&p, sizeof(float) * m * d);
        if (e != cudaSuccess) {
            delete h;
            KNN_CUDA_CHECK(e);
        }
        h->dR = p;
        h->owned = true;
        e = cudaMemcpy(p, references, sizeof(float) * m * d, cudaMemcpyHostToDevice);
        if (e != cudaSuccess) {
            delete h;
            KNN_CUDA_CHECK(e);
        }
        try {
            std::lock_guard<std::mutex> lock(ctx.mu);
            prepare_index(ctx, h);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

knn_b200_status knn_b200_index_create_device(const float* d_references, int64_t m, int32_t d,
                                             int64_t index_base, const knn_b200_options* opt,
                                             knn_b200_index** out) {
    return guarded([&] {
        knn_b200_options tmp;
        const knn_b200_options& o = opts_or_default(opt, tmp);
        if (!out) throw InvalidArgument("knn_b200_index_create: null out");
        check_point_set(d_references, m, d, false);
        DeviceContext& ctx = context_for(o.device);
        KNN_CUDA_CHECK(cudaSetDevice(ctx.device));
        std::lock_guard<std::mutex> lock(ctx.mu);
        check_finite_device(ctx.stream, d_references, m, d, nullptr);
        auto* h = new knn_b200_index();
        h->device = ctx.device;
        h->dR = d_references;
        h->owned = false;
        h->m = m;
        h->d = d;
        h->base = index_base;
        try {
            prepare_index(ctx, h);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

knn_b200_status knn_b200_index_search(knn_b200_index* index, const float* queries, int64_t n,
                                      int32_t k, int32_t metric, const knn_b200_options* opt,
                                      float* out_dist, int64_t* out_idx) {
    return guarded([&] {
        if (!index) throw InvalidArgument("knn_b200_index_search: null index");
        knn_b200_options tmp;
        const knn_b200_options& o = opts_or_default(opt, tmp);
        if (metric == kMahalanobis)
            throw InvalidArgument("knn_b200_index_search: whiten inputs for Mahalanobis");
        check_point_set(queries, n, index->d, true);
        check_search(index->d, index->d, index->m, k, o, metric);
        DeviceContext& ctx = context_for(index->device);
        std::lock_guard<std::mutex> hl(index->mu);
        std::lock_guard<std::mutex> lock(ctx.mu);
        KNN_CUDA_CHECK(cudaSetDevice(ctx.device));
        cudaStream_t s = o.stream ? static_cast<cudaStream_t>(o.stream) : ctx.stream;
        ctx.bind(s);
        Sizer sz;
        sz.take<float>(static_cast<size_t>(n) * index->d);
        sz.take<float>(static_cast<size_t>(n) * k);
        sz.take<int64_t>(static_cast<size_t>(n) * k);
        ctx.s->io.reserve(sz.used + 256);
        Carver cv{static_cast<char*>(ctx.s->io.base())};
        float* dQ = cv.take<float>(static_cast<size_t>(n) * index->d);
        float* dO = cv.take<float>(static_cast<size_t>(n) * k);
        int64_t* dI = cv.take<int64_t>(static_cast<size_t>(n) * k);
        KNN_CUDA_CHECK(cudaMemcpyAsync(dQ, queries, sizeof(float) * n * index->d,
                                       cudaMemcpyHostToDevice, s));
        search_device(ctx, s, dQ, n, index->dR, index->m, index->d, k, metric, o.path,
                      o.raw_keys, index->base, dO, dI, index_refs(index, n, k, metric, o.path));
        KNN_CUDA_CHECK(
            cudaMemcpyAsync(out_dist, dO, sizeof(float) * n * k, cudaMemcpyDeviceToHost, s));
        KNN_CUDA_CHECK(
            cudaMemcpyAsync(out_idx, dI, sizeof(int64_t) * n * k, cudaMemcpyDeviceToHost, s));
        KNN_CUDA_CHECK(cudaStreamSynchronize(s));
    });
}

knn_b200_status knn_b200_index_search_device(knn_b200_index* index, const float* d_queries,
                                             int64_t n, int32_t k, int32_t metric,
                                             const knn_b200_options* opt, float* d_out_dist,
                                             int64_t* d_out_idx) {
    return guarded([&] {
        if (!index) throw InvalidArgument("knn_b200_index_search: null index");
        knn_b200_options tmp;
        const knn_b200_options& o = opts_or_default(opt, tmp);
        if (metric == kMahalanobis)
            throw InvalidArgument("knn_b200_index_search: whiten inputs for Mahalanobis");
        check_point_set(d_queries, n, index->d, false);
        check_search(index->d, index->d, index->m, k, o, metric);
        DeviceContext& ctx = context_for(index->device);
        std::lock_guard<std::mutex> hl(index->mu);
        std::lock_guard<std::mutex> lock(ctx.mu);
        KNN_CUDA_CHECK(cudaSetDevice(ctx.device));
        cudaStream_t s = o.stream ? static_cast<cudaStream_t>(o.stream) : ctx.stream;
        ctx.bind(s);
        if (!o.stream) check_finite_device(s, d_queries, n, index->d, nullptr);
        search_device(ctx, s, d_queries, n, index->dR, index->m, index->d, k, metric, o.path,
                      o.raw_keys, index->base, d_out_dist, d_out_idx,
                      index_refs(index, n, k, metric, o.path));
        if (!o.stream) KNN_CUDA_CHECK(cudaStreamSynchronize(s));
    });
}

void knn_b200_index_destroy(knn_b200_index* index) { delete index; }

int knn_b200_last_fallback_count(int device) {
    try {
        DeviceContext& ctx = context_for(device);
        std::lock_guard<std::mutex> lock(ctx.mu);
        const Scratch* sc = ctx.last;
        if (!sc) return 0;
        if (sc->fb_on_device) {  // resolved on the device by the last search
            int v = 0;
            KNN_CUDA_CHECK(cudaSetDevice(ctx.device));
            KNN_CUDA_CHECK(cudaDeviceSynchronize());
            KNN_CUDA_CHECK(cudaMemcpy(&v, sc->fb_dev, sizeof(int), cudaMemcpyDeviceToHost));
            return v;
        }
        return sc->last_fallbacks;
    } catch (...) {
        return -1;
    }
}

knn_b200_status knn_b200_merge_device(const float* d_part_keys, const int64_t* d_part_idx,
                                      int32_t parts, int64_t n, int32_t k, int32_t metric,
                                      void* stream, float* d_out_dist, int64_t* d_out_idx) {
    return guarded([&] {
        if (parts <= 0 || n <= 0 || k <= 0)
            throw InvalidArgument("knn_b200_merge_device: parts, n and k must be >= 1");
        DeviceContext& ctx = context_for(-1);
        std::lock_guard<std::mutex> lock(ctx.mu);
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : ctx.stream;
        ctx.bind(s);
        MergeArgs mg{};
        mg.part_key = d_part_keys;
        mg.part_idx = d_part_idx;
        mg.parts = parts;
        mg.n = n;
        mg.k = k;
        mg.metric = metric == kMahalanobis ? kL2 : metric;
        mg.finalize = 1;
        mg.out_key = d_out_dist;
        mg.out_idx = d_out_idx;
        if (k > 1024) {
            Sizer sz;
            sz.take<float>(static_cast<size_t>(n) * k);
            sz.take<int64_t>(static_cast<size_t>(n) * k);
            ctx.s->arena.reserve(sz.used + 256);
            Carver cv{static_cast<char*>(ctx.s->arena.base())};
            mg.glist_key = cv.take<float>(static_cast<size_t>(n) * k);
            mg.glist_idx = cv.take<int64_t>(static_cast<size_t>(n) * k);
        }
        launch_merge(mg, s);
        if (!stream) KNN_CUDA_CHECK(cudaStreamSynchronize(s));
    });
}

}  // extern "C"
