// exact_kernel.cuh -- host interface of the exact SIMT path.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace knnb200 {

struct ExactArgs {
    const float* Q;          // query rows (row i of the search = Q row qlist ? qlist[i] : i)
    const float* R;          // m x d
    int64_t n, m;            // n: queries (the maximum when qcount is set)
    int d, k;
    int ntiles;              // reference tiles per query block (exact_plan)
    const int* qlist;        // nullable: query i's row in Q and in the outputs
    const int* qcount;       // nullable: device-side query count (<= n)
    int64_t index_base;      // added to every emitted index
    int raw_keys;            // 1: outputs keep raw keys (no finalize)
    float* out_key;          // final outputs, n x k rows
    int64_t* out_idx;
    // Stream-K segments (CTA c, query block b) that share a block write their
    // raw lists to slot c + b of [slots][128][k]; a block with one segment is
    // emitted final by the exact kernel, the others by merge_exact.
    float* part_key;
    int64_t* part_idx;
    float* glist_key;        // global list scratch when k is too large for smem
    int32_t* glist_idx;
    float* mglist_key;       // merge list scratch (n x k) when k > 2048
    int64_t* mglist_idx;
    int max_ctas;            // set by launch_exact (grid of the exact kernel)
    int min_tiles;           // set by launch_exact: reference tiles per CTA at least (0: 8)
    // threshold-log mode (large k, exact_large.cu): instead of lists, every key
    // <= t0[q * t0_stride] is appended as {key, index bits} to the segment's
    // log vlog[slot][128][CV] (column order), its length to vlog_n[slot][128]
    const float* t0;
    int t0_stride;
    float2* vlog;
    int* vlog_n;
    int CV;
};

// Stream-K split of the exact path, a pure function of the query count so the
// device can re-derive it from a device-side count: G CTAs (<= max_ctas, >= 8
// tiles each) own contiguous ranges of the (query block, tile) units.
struct ExactSplit {
    int64_t units;
    int64_t G;
    __host__ __device__ int64_t start(int64_t c) const { return c * units / G; }
    __host__ __device__ int64_t cta_of(int64_t x) const { return ((x + 1) * G + units - 1) / units - 1; }
};
__host__ __device__ inline ExactSplit exact_split(int64_t n, int ntiles, int max_ctas, int min_tiles = 8) {
    const int64_t nqb = (n + 127) / 128;
    ExactSplit s;
    s.units = nqb * ntiles;
    const int64_t per = min_tiles > 8 ? min_tiles : 8;
    const int64_t by_work = s.units / per > 1 ? s.units / per : 1;
    s.G = by_work < max_ctas ? by_work : max_ctas;
    return s;
}

// Resident CTAs of the exact kernel (grid size) and reference tiles per block.
int exact_max_ctas(int k, bool smem_lists);
int exact_ntiles(int64_t m);
// partial-list slots for up to n queries: G + query blocks
int64_t exact_slots(int64_t n, int ntiles, int max_ctas);
// exact kernel (grid = max CTAs; the CTAs past the split's G exit) followed by
// merge_exact when some block spans several CTAs (always when qcount is set)
void launch_exact(int metric, const ExactArgs& a, cudaStream_t stream);
// the threshold-log pass of the exact path (no merge; a.vlog etc. set)
void launch_exact_log(int metric, const ExactArgs& a, cudaStream_t stream);
int exact_log_max_ctas();  // grid of the threshold-log pass
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
