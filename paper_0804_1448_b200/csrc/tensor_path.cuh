// tensor_path.cuh -- tcgen05 candidate path (fp16 GEMM form + exact re-rank).
#pragma once

#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <stddef.h>
#include <stdint.h>

namespace knnb200 {

struct DeviceContext;

bool tensor_path_supported(int64_t n, int64_t m, int d, int k);

void run_tensor_path(DeviceContext& ctx, cudaStream_t stream, const float* dQ, int64_t n,
                     const float* dR, int64_t m, int d, int k, int raw_keys, int64_t index_base,
                     float* d_out, int64_t* d_idx);

// Reference-side state of the tensor path (fp16 copy with folded norms,
// centre/scale, rounding radii), built once per reference set and reusable by
// any number of query searches (index handles, the pipelined host API).
struct TensorRefs {
    const float* dR = nullptr;  // original FP32 references (exact re-rank)
    int64_t m = 0, m_pad = 0;
    int d = 0;
    __half* Rh = nullptr;
    float* rnorm = nullptr;
    float* mu = nullptr;
    float* scale = nullptr;
    unsigned* gmax = nullptr;
};
size_t tensor_refs_bytes(int64_t m, int d);
void tensor_prep_refs(cudaStream_t stream, const float* dR, int64_t m, int d, void* mem,
                      TensorRefs& out);

// Deferred certification fallbacks: failed queries are appended (index +
// offset) to a device list instead of being recomputed inside the search.
struct FallbackSink {
    int* count;
    int* list;
    int offset;
};

// margin: large-k threshold target, T0 ~ the (margin*k)-th smallest A.
void tensor_search(DeviceContext& ctx, cudaStream_t stream, const TensorRefs& refs,
                   const float* dQ, int64_t n, int k, int raw_keys, int64_t index_base,
                   float* d_out, int64_t* d_idx, const FallbackSink* sink = nullptr,
                   int margin = 3);

// Resolve the certification fallbacks recorded in fb ({count, query list}) of
// a search over dQ (n rows) on the device: the exact kernel over the list
// (fb_pk / fb_pi: fallback_part_elems(n, m, k) partial-list slots; fb_gk /
// fb_gi: fallback_glist_elems(k) list scratch, k > 128).
size_t fallback_part_elems(int64_t n, int64_t m, int k);
size_t fallback_glist_elems(int k);
void tensor_resolve_fallbacks(DeviceContext& ctx, cudaStream_t stream, const TensorRefs& refs,
                              const float* dQ, int64_t n, int k, int raw_keys, int64_t index_base,
                              float* d_out, int64_t* d_idx, int* fb, float* fb_pk, int64_t* fb_pi,
                              float* fb_gk, int32_t* fb_gi);

}  // namespace knnb200
