// merge_kernel.cu -- merge per-part top-k lists into the final top-k.
//
// Used for (a) the stream-K parts of one GPU's exact search (a query block
// spread over several CTAs) and (b) the shard merge of a reference-sharded
// multi-GPU search after the all-gather.  Each part's list
// is the top-k of a disjoint reference range, sorted under the (key, index) order
// (topk.cpp:11-13); the top-k of the union equals the top-k of the union of
// the part top-ks, so the result is bitwise independent of how the
// reference set was split.
#include "common.cuh"
#include "exact_kernel.cuh"
#include "profile.cuh"
#include "warp_list.cuh"

namespace knnb200 {

namespace {

constexpr int WARPS = 4;

template <bool SMEM_LISTS>
__global__ void __launch_bounds__(WARPS * 32) merge_kernel(MergeArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int64_t q = static_cast<int64_t>(blockIdx.x) * WARPS + warp;
    if (q >= a.n) return;
    const int k = a.k;

    float* lk;
    int64_t* li;
    if constexpr (SMEM_LISTS) {
        lk = reinterpret_cast<float*>(smem_raw) + warp * k;
        li = reinterpret_cast<int64_t*>(reinterpret_cast<float*>(smem_raw) + WARPS * k +
                                        (WARPS * k & 1)) + warp * k;
    } else {
        lk = a.glist_key + q * k;
        li = a.glist_idx + q * k;
    }
    WarpList<int64_t> L{lk, li, k};

    // part 0 is already a sorted top-k list: adopt it as the initial list
    const size_t stride = static_cast<size_t>(a.n) * k;
    for (int t = lane; t < k; t += 32) {
        lk[t] = a.part_key[q * k + t];
        li[t] = a.part_idx[q * k + t];
    }
    __syncwarp();

    for (int p = 1; p < a.parts; ++p) {
        const float* pk = a.part_key + p * stride + q * k;
        const int64_t* pi = a.part_idx + p * stride + q * k;
        for (int t0 = 0; t0 < k; t0 += 128) {
            float ck[4];
            int64_t ci[4];
#pragma unroll
            for (int s = 0; s < 4; ++s) {
                const int t = t0 + lane + 32 * s;
                ck[s] = t < k ? pk[t] : kInf;
                ci[s] = t < k ? pi[t] : kSentinelIdx;
            }
            // sorted parts: once this chunk's smallest fails the threshold the
            // rest of the part fails too
            float tk;
            int64_t ti;
            L.threshold(tk, ti);
            const float first_k = __shfl_sync(0xffffffffu, ck[0], 0);
            const int64_t first_i = __shfl_sync(0xffffffffu, ci[0], 0);
            if (!pair_less(first_k, first_i, tk, ti)) break;
            L.offer<4>(ck, ci, lane);
        }
    }
    __syncwarp();
    if (a.finalize) finalize_list(lk, li, k, a.metric, lane);
    for (int t = lane; t < k; t += 32) {
        a.out_key[q * k + t] = lk[t];
        a.out_idx[q * k + t] = li[t];
    }
}

}  // namespace

void launch_merge(const MergeArgs& a, cudaStream_t stream) {
    const bool smem_lists = a.glist_key == nullptr;
    const size_t smem =
        smem_lists ? static_cast<size_t>(WARPS) * a.k * (sizeof(float) + sizeof(int64_t)) + 8 : 0;
    const unsigned grid = static_cast<unsigned>((a.n + WARPS - 1) / WARPS);
    if (smem_lists) {
        KNN_CUDA_CHECK(cudaFuncSetAttribute(merge_kernel<true>,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            static_cast<int>(smem)));
        ProfileScope ps(stream, "merge_kernel");
        merge_kernel<true><<<grid, WARPS * 32, smem, stream>>>(a);
    } else {
        ProfileScope ps(stream, "merge_kernel_glist");
        merge_kernel<false><<<grid, WARPS * 32, 0, stream>>>(a);
    }
    KNN_LAUNCH_CHECK();
}

}  // namespace knnb200
