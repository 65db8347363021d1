// engine.cu -- search orchestration on one device.
//
// The reference's bf_knn (src/bruteforce.cpp:42-100) processes queries in
// chunks of chunk_size rows with an OpenMP fork/join per chunk and a
// chunk x m double scratch.  Here one search is a short fixed sequence of
// kernel launches on one stream with all scratch carved from a grow-only
// per-device arena:
//   exact path   exact_knn_kernel (fused keys + top-k per reference split)
//                [+ merge_kernel when the reference axis was split]
//   tensor path  see tensor_kernel.cu (prep -> tcgen05 candidates ->
//                exact re-rank -> exact fallback for uncertified queries)
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <memory>

#include "common.cuh"
#include "engine.cuh"
#include "exact_kernel.cuh"
#include "tensor_path.cuh"

namespace knnb200 {

DeviceArena::~DeviceArena() {
    if (base_) cudaFree(base_);
    for (void* p : retired_) cudaFree(p);
}

namespace {
thread_local bool t_capturing = false;  // the bound stream is being captured into a graph

// queries per tensor-path search of a device-pointer call (multiple of the
// 256-query pair; dev knob KNN_B200_TENSOR_CHUNK)
int64_t tensor_query_chunk() {
    static const int64_t v = [] {
        const char* e = std::getenv("KNN_B200_TENSOR_CHUNK");
        const int64_t c = e ? std::max<int64_t>(256, std::atoll(e)) : int64_t{1} << 18;
        return (c + 255) / 256 * 256;
    }();
    return v;
}

// fb[1] = (first ? 0 : fb[1]) + fb[0]: the fallback count summed over query chunks
__global__ void sum_count_kernel(int* fb, bool first) {
    if (threadIdx.x == 0) fb[1] = (first ? 0 : fb[1]) + fb[0];
}
}

void DeviceArena::reserve(size_t bytes) {
    if (t_capturing) captured_ = true;
    if (bytes <= cap_) return;
    if (t_capturing)
        throw CudaError("knn_b200: scratch would have to grow during CUDA graph capture; run the "
                        "same search once outside the capture first");
    const size_t want = std::max(bytes, cap_ + cap_ / 2);
    if (base_) {
        if (captured_) {
            retired_.push_back(base_);  // a captured graph may still replay on it
        } else {
            KNN_CUDA_CHECK(cudaDeviceSynchronize());
            KNN_CUDA_CHECK(cudaFree(base_));
        }
        base_ = nullptr;
        cap_ = 0;
    }
    KNN_CUDA_CHECK(cudaMalloc(&base_, want));
    cap_ = want;
}

Scratch::~Scratch() {
    if (fb_dev) cudaFree(fb_dev);
}

Scratch& DeviceContext::bind(cudaStream_t st) {
    auto& slot = scratch[st];
    if (!slot) slot = std::make_unique<Scratch>();
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    KNN_CUDA_CHECK(cudaStreamIsCapturing(st, &cs));
    t_capturing = cs != cudaStreamCaptureStatusNone;
    if (!slot->fb_dev && !t_capturing) KNN_CUDA_CHECK(cudaMalloc(&slot->fb_dev, 2 * sizeof(int)));
    s = slot.get();
    last = s;
    return *s;
}

DeviceContext& context_for(int device) {
    static std::mutex registry_mu;
    static std::map<int, std::unique_ptr<DeviceContext>> registry;
    if (device < 0) KNN_CUDA_CHECK(cudaGetDevice(&device));
    std::lock_guard<std::mutex> lock(registry_mu);
    auto& slot = registry[device];
    if (!slot) {
        slot = std::make_unique<DeviceContext>();
        slot->device = device;
        KNN_CUDA_CHECK(cudaSetDevice(device));
        // stream-ordered allocations (cudaMallocAsync) stay cached in the
        // device's default pool across synchronisations instead of being
        // unmapped at every one (release threshold 0) and re-mapped next call
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
            uint64_t keep = UINT64_MAX;
            KNN_CUDA_CHECK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
        }
        KNN_CUDA_CHECK(cudaStreamCreateWithFlags(&slot->stream, cudaStreamNonBlocking));
        KNN_CUDA_CHECK(cudaStreamCreateWithFlags(&slot->copy_stream, cudaStreamNonBlocking));
        for (auto& e : slot->ev) KNN_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    return *slot;
}

SearchPlan plan_search(int64_t n, int64_t m, int d, int k, int metric, int path) {
    SearchPlan p{};
    p.path = 1;
    if (path != 1 && metric == kL2 && tensor_path_supported(n, m, d, k)) p.path = 2;
    if (path == 2 && p.path != 2 && metric == kL2 && !tensor_path_supported(n, m, d, k))
        p.path = 1;  // TENSOR requested for an unsupported shape: exact gives identical results
    return p;
}

// the list path of the exact kernel (any k): lists in shared memory up to
// k = 128, global memory beyond
void run_exact_lists(DeviceContext& ctx, cudaStream_t stream, const float* dQ, int64_t n,
                     const float* dR, int64_t m, int d, int k, int metric, int raw_keys,
                     int64_t index_base, float* d_out, int64_t* d_idx) {
    const bool big_k = static_cast<size_t>(k) > exact_smem_list_limit_k();
    ExactArgs a{};
    a.Q = dQ;
    a.R = dR;
    a.n = n;
    a.m = m;
    a.d = d;
    a.k = k;
    a.ntiles = exact_ntiles(m);
    a.index_base = index_base;
    a.raw_keys = raw_keys;
    a.out_key = d_out;
    a.out_idx = d_idx;
    const int max_ctas = exact_max_ctas(k, !big_k);
    const size_t part = static_cast<size_t>(exact_slots(n, a.ntiles, max_ctas)) *
                        exact_queries_per_cta() * k;
    const size_t lists = static_cast<size_t>(max_ctas) * exact_queries_per_cta() * k;
    Sizer sz;
    sz.take<float>(part);
    sz.take<int64_t>(part);
    if (big_k) {
        sz.take<float>(lists);
        sz.take<int32_t>(lists);
    }
    if (k > 2048) {
        sz.take<float>(static_cast<size_t>(n) * k);
        sz.take<int64_t>(static_cast<size_t>(n) * k);
    }
    ctx.s->arena.reserve(sz.used + 256);
    Carver cv{static_cast<char*>(ctx.s->arena.base())};
    a.part_key = cv.take<float>(part);
    a.part_idx = cv.take<int64_t>(part);
    if (big_k) {
        a.glist_key = cv.take<float>(lists);
        a.glist_idx = cv.take<int32_t>(lists);
    }
    if (k > 2048) {
        a.mglist_key = cv.take<float>(static_cast<size_t>(n) * k);
        a.mglist_idx = cv.take<int64_t>(static_cast<size_t>(n) * k);
    }
    launch_exact(metric, a, stream);
}

// exact path: the threshold-log path for 128 < k <= 1024 on large reference
// sets (exact_large.cu), the list path otherwise (dev knob
// KNN_B200_EXACT_LARGE=0 forces the list path)
static void run_exact(DeviceContext& ctx, cudaStream_t stream, const float* dQ, int64_t n,
                      const float* dR, int64_t m, int d, int k, int metric, int raw_keys,
                      int64_t index_base, float* d_out, int64_t* d_idx) {
    static const bool large_ok = [] {
        const char* e = std::getenv("KNN_B200_EXACT_LARGE");
        return !(e && std::atoi(e) == 0);
    }();
    if (large_ok && exact_large_applies(m, k)) {
        run_exact_large(ctx, stream, dQ, n, dR, m, d, k, metric, raw_keys, index_base, d_out, d_idx);
        return;
    }
    run_exact_lists(ctx, stream, dQ, n, dR, m, d, k, metric, raw_keys, index_base, d_out, d_idx);
}

void search_device(DeviceContext& ctx, cudaStream_t stream, const float* dQ, int64_t n,
                   const float* dR, int64_t m, int d, int k, int metric, int path,
                   int raw_keys, int64_t index_base, float* d_out, int64_t* d_idx,
                   const TensorRefs* refs) {
    const SearchPlan plan = plan_search(n, m, d, k, metric, path);
    const int64_t qchunk = tensor_query_chunk();
    if (plan.path == 2 && n > qchunk) {
        // query chunks bound the per-search scratch (the group logs grow as
        // n x parts x log capacity); the reference set is prepared once and
        // the fallback count summed over the chunks on the device
        TensorRefs local;
        const TensorRefs* rp = refs;
        if (!rp) {
            ctx.s->refs.reserve(tensor_refs_bytes(m, d));
            tensor_prep_refs(stream, dR, m, d, ctx.s->refs.base(), local);
            rp = &local;
        }
        int* fb = ctx.s->fb_dev;
        for (int64_t q0 = 0; q0 < n; q0 += qchunk) {
            const int64_t nq = std::min(qchunk, n - q0);
            tensor_search(ctx, stream, *rp, dQ + q0 * d, nq, k, raw_keys, index_base, d_out + q0 * k,
                          d_idx + q0 * k);
            if (fb) {
                sum_count_kernel<<<1, 32, 0, stream>>>(fb, q0 == 0);
                KNN_LAUNCH_CHECK();
            }
        }
        if (fb) KNN_CUDA_CHECK(cudaMemcpyAsync(fb, fb + 1, sizeof(int), cudaMemcpyDeviceToDevice, stream));
        return;
    }
    if (plan.path == 2) {
        if (refs)  // reference set already prepared (index handle)
            tensor_search(ctx, stream, *refs, dQ, n, k, raw_keys, index_base, d_out, d_idx);
        else
            run_tensor_path(ctx, stream, dQ, n, dR, m, d, k, raw_keys, index_base, d_out, d_idx);
        return;
    }
    run_exact(ctx, stream, dQ, n, dR, m, d, k, metric, raw_keys, index_base, d_out, d_idx);
}

}  // namespace knnb200
