// tensor_path.cuh -- tcgen05 candidate path (fp16 GEMM form + exact re-rank).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace knnb200 {

struct DeviceContext;

bool tensor_path_supported(int64_t n, int64_t m, int d, int k);

// margin: large-k threshold target, T0 ~ the (margin*k)-th smallest A; the
// large-k certification fallback retries once (retry = true) from fresh seed
// tiles before the exact path.
void run_tensor_path(DeviceContext& ctx, cudaStream_t stream, const float* dQ, int64_t n,
                     const float* dR, int64_t m, int d, int k, int raw_keys, int64_t index_base,
                     float* d_out, int64_t* d_idx, int margin = 2, bool retry = false);

// exact path on a subset of queries (certification fallback), defined in engine.cu
void run_exact_subset(DeviceContext& ctx, cudaStream_t stream, const float* dQ, int64_t n,
                      const float* dR, int64_t m, int d, int k, int raw_keys, int64_t index_base,
                      float* d_out, int64_t* d_idx);

}  // namespace knnb200
