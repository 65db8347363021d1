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
    int64_t units;           // stream-K work units: query blocks x reference tiles
    int ntiles;              // reference tiles per query block
    int ctas;                // grid size (each CTA owns a contiguous unit range)
    int parts;               // output slots per query (max CTAs sharing a query block)
    int64_t index_base;      // added to every emitted index
    float* out_key;          // [parts][n][k]
    int64_t* out_idx;        // [parts][n][k]
    int finalize;            // 1: out_key = finalized distance (parts == 1 only)
    float* glist_key;        // global list scratch when k is too large for smem
    int32_t* glist_idx;
};

// Work split of the exact kernel over the GPU: fills units/ntiles/ctas/parts.
void exact_plan(ExactArgs& a, bool smem_lists);
void launch_exact(int metric, const ExactArgs& a, cudaStream_t stream);
size_t exact_smem_list_limit_k();
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
