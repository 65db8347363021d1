// exact_kernel.cuh -- host interface of the exact SIMT path.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace knnb200 {

struct ExactArgs {
    const float* Q;          // n x d
    const float* R;          // m x d
    int64_t n, m;
    int d, k;
    int64_t split_len;       // references per blockIdx.y split (>= k)
    int splits;
    int64_t index_base;      // added to every emitted index
    float* out_key;          // [splits][n][k]
    int64_t* out_idx;        // [splits][n][k]
    int finalize;            // 1: out_key = finalized distance (splits == 1 only)
    float* glist_key;        // global list scratch when k is too large for smem
    int32_t* glist_idx;
};

void launch_exact(int metric, const ExactArgs& a, cudaStream_t stream);
size_t exact_smem_list_limit_k();
size_t exact_cta_count(int64_t n, int splits);
int exact_queries_per_cta();

struct MergeArgs {
    const float* part_key;   // [parts][n][k] raw keys, each part sorted ascending
    const int64_t* part_idx;
    int parts;
    int64_t n;
    int k;
    int metric;
    int finalize;
    float* out_key;          // n x k
    int64_t* out_idx;
    float* glist_key;        // scratch for k > smem limit (n x k), or nullptr
    int64_t* glist_idx;
};

void launch_merge(const MergeArgs& a, cudaStream_t stream);

}  // namespace knnb200
