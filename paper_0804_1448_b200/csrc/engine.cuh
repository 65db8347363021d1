// engine.cuh -- host-side engine: device contexts, workspaces, search plans.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <memory>
#include <mutex>
#include <vector>

namespace knnb200 {

// Grow-only device scratch arena.  Carves aligned slices out of one
// allocation so a search does a single cudaMalloc at most.  A block that a
// captured CUDA graph may reference is never freed while the context lives
// (growing retires it instead), and the arena cannot grow during a capture.
class DeviceArena {
public:
    ~DeviceArena();
    void reserve(size_t bytes);
    void* base() const { return base_; }
    void mark_captured() { captured_ = true; }

private:
    void* base_ = nullptr;
    size_t cap_ = 0;
    bool captured_ = false;
    std::vector<void*> retired_;
};

// Per-stream scratch of a context: searches on different streams run
// concurrently and must not share scratch; searches on one stream are
// ordered by the stream, so they reuse it.
struct Scratch {
    DeviceArena arena;       // per-search scratch
    DeviceArena io;          // host-API staging of inputs / outputs
    DeviceArena refs;        // tensor path: prepared reference set of a one-shot search
    DeviceArena coll;        // multi-GPU: local and all-gathered shard lists
    DeviceArena xl;          // exact large-k selection (also the tensor path's large-k fallback)
    int last_fallbacks = 0;  // tensor path: queries re-run on the exact kernel
    int* fb_dev = nullptr;   // ... the same count, when resolved on the device
                             // ([0] the count, [1] a running sum over query chunks)
    bool fb_on_device = false;
    ~Scratch();
};

struct Carver {
    char* p;
    size_t used = 0;
    template <typename T>
    T* take(size_t count) {
        used = (used + 255) & ~static_cast<size_t>(255);
        T* out = reinterpret_cast<T*>(p + used);
        used += count * sizeof(T);
        return out;
    }
};

// Bytes a Carver needs for the given take() sizes (same 256 B alignment).
struct Sizer {
    size_t used = 0;
    template <typename T>
    void take(size_t count) {
        used = (used + 255) & ~static_cast<size_t>(255);
        used += count * sizeof(T);
    }
};

struct DeviceContext {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t copy_stream = nullptr;   // host API: H2D / D2H overlapped with compute
    cudaEvent_t ev[16] = {};              // host API pipeline events
    std::vector<cudaEvent_t> pipe_ev;     // per-chunk events of the pipelined host search
    std::mutex mu;           // serializes the host-side enqueue of searches
    std::map<cudaStream_t, std::unique_ptr<Scratch>> scratch;
    Scratch* s = nullptr;     // scratch of the stream bound by the current call
    Scratch* last = nullptr;  // scratch of the last search (fallback count)
    // Select (create) the scratch of `stream` for the calling search (under mu).
    Scratch& bind(cudaStream_t stream);
};

DeviceContext& context_for(int device);  // device < 0: current device

struct SearchPlan {
    int path;       // 1 exact, 2 tensor
};

struct TensorRefs;

// Core device search.  All pointers are device pointers.  Output: finalized
// distances (or raw keys when raw_keys) and global indices (index_base + j).
// refs: the tensor path's prepared reference set (index handles), optional.
// exact path pieces (engine.cu, exact_large.cu)
void run_exact_lists(DeviceContext& ctx, cudaStream_t stream, const float* dQ, int64_t n,
                     const float* dR, int64_t m, int d, int k, int metric, int raw_keys,
                     int64_t index_base, float* d_out, int64_t* d_idx);
bool exact_large_applies(int64_t m, int k);
// (qlist, qcount): device-side query list (positions -> rows of dQ and of the
// outputs), e.g. the tensor path's certification fallback; n = list capacity
void run_exact_large(DeviceContext& ctx, cudaStream_t stream, const float* dQ, int64_t n,
                     const float* dR, int64_t m, int d, int k, int metric, int raw_keys,
                     int64_t index_base, float* d_out, int64_t* d_idx, const int* qlist = nullptr,
                     const int* qcount = nullptr);

void search_device(DeviceContext& ctx, cudaStream_t stream, const float* dQ, int64_t n,
                   const float* dR, int64_t m, int d, int k, int metric, int path,
                   int raw_keys, int64_t index_base, float* d_out, int64_t* d_idx,
                   const TensorRefs* refs = nullptr);

SearchPlan plan_search(int64_t n, int64_t m, int d, int k, int metric, int path);

// PointSet's value check (point_set.hpp:27-31) on device rows: throws
// InvalidArgument naming the first non-finite coordinate (capi.cu).
void check_finite_device(cudaStream_t s, const float* X, int64_t rows, int64_t d,
                         unsigned long long* dbad);

}  // namespace knnb200
