// common.cuh -- shared definitions for the B200 brute-force kNN engine.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

namespace knnb200 {

enum Metric : int { kL2 = 0, kL1 = 1, kLinf = 2, kMahalanobis = 3 };

constexpr int kSmCount = 148;                  // B200: 2 dies x 74 SMs
constexpr float kInf = __builtin_huge_valf();
constexpr int64_t kSentinelIdx = INT64_MAX;    // empty list slot, sorts last

// Host-side error types mapped to ABI status codes by capi.cpp.
struct InvalidArgument : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct OutOfMemory : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct NcclError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// The C ABI's error convention (capi.cu): run `body`, map exceptions to
// status codes, keep the message for knn_b200_last_error() (thread-local).
void set_last_error(const std::string& msg);
template <typename F>
int abi_guarded(F&& body) {
    try {
        set_last_error("");
        body();
        return 0;                                               // KNN_B200_OK
    } catch (const InvalidArgument& e) {
        set_last_error(e.what());
        return 1;                                               // KNN_B200_EINVAL
    } catch (const OutOfMemory& e) {
        set_last_error(e.what());
        return 2;                                               // KNN_B200_ENOMEM
    } catch (const CudaError& e) {
        set_last_error(e.what());
        return 3;                                               // KNN_B200_ECUDA
    } catch (const NcclError& e) {
        set_last_error(e.what());
        return 4;                                               // KNN_B200_ENCCL
    } catch (const std::bad_alloc&) {
        set_last_error("host allocation failed");
        return 2;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return 5;                                               // KNN_B200_EINTERNAL
    }
}

void note_launch(int count = 1);  // launch accounting (capi.cpp)

#define KNN_CUDA_CHECK(expr)                                                              \
    do {                                                                                  \
        cudaError_t err_ = (expr);                                                        \
        if (err_ != cudaSuccess) {                                                        \
            if (err_ == cudaErrorMemoryAllocation)                                        \
                throw ::knnb200::OutOfMemory(std::string("CUDA out of memory: ") + #expr); \
            throw ::knnb200::CudaError(std::string(#expr) + ": " +                        \
                                       cudaGetErrorString(err_));                         \
        }                                                                                 \
    } while (0)

#define KNN_LAUNCH_CHECK()                                  \
    do {                                                    \
        ::knnb200::note_launch();                           \
        KNN_CUDA_CHECK(cudaGetLastError());                 \
    } while (0)

// ---------------------------------------------------------------- device ----
// (key, index) lexicographic order of the reference's selection
// (topk.cpp:11-13).  Sentinel entries are (+inf, INT64_MAX) and sort last.
__device__ __forceinline__ bool pair_less(float ka, int64_t ia, float kb, int64_t ib) {
    return ka < kb || (ka == kb && ia < ib);
}

// One coordinate step of a metric key, in the reference's fixed coordinate
// order (metric.hpp:22-44).  L2 uses one rounding per step pair:
// t = q - r (rn), acc = fma(t, t, acc) (rn).  Every code path that produces an
// exact key (SIMT kernel, re-rank) uses exactly this function, so a pair's key
// is bitwise identical whichever path computed it.
template <int M>
__device__ __forceinline__ float key_step(float acc, float q, float r) {
    const float t = __fsub_rn(q, r);
    if constexpr (M == kL2) {
        return __fmaf_rn(t, t, acc);
    } else if constexpr (M == kL1) {
        return __fadd_rn(acc, fabsf(t));
    } else {
        return fmaxf(acc, fabsf(t));  // = (|t| > acc ? |t| : acc) on finite keys
    }
}

template <int M>
__device__ __forceinline__ float finalize_key(float key) {
    if constexpr (M == kL2) return __fsqrt_rn(key);
    return key;
}

__device__ __forceinline__ float finalize_key_rt(int metric, float key) {
    return metric == kL2 ? __fsqrt_rn(key) : key;
}

}  // namespace knnb200
