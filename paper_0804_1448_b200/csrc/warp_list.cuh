// warp_list.cuh -- warp-cooperative sorted top-k list.
//
// Replaces the reference's per-row select_k_smallest (src/topk.cpp:17-33:
// nth_element + sort over a materialised m-long row) with a streaming
// structure: a list of the k best (key, index) pairs seen so far, kept sorted
// ascending under the (key, index) order, stored in shared (or global) memory
// and updated by one warp.  Candidates are filtered against the list's k-th
// entry (the running threshold) before any insertion, so after the first few
// tiles almost every candidate is rejected with one compare.
//
// Layout: entry i of a list lives at key[i], idx[i] (i < k).  Unfilled slots
// hold the sentinel (+inf, INT64_MAX), so the threshold is always key[k-1].
#pragma once

#include "common.cuh"

namespace knnb200 {

template <typename IdxT>
__device__ __forceinline__ IdxT sentinel_of() {
    return sizeof(IdxT) == 8 ? static_cast<IdxT>(kSentinelIdx) : static_cast<IdxT>(0x7fffffff);
}

template <typename IdxT>
struct WarpList {
    float* key;  // k entries
    IdxT* idx;   // k entries
    int k;

    __device__ __forceinline__ void init(int lane) {
        for (int i = lane; i < k; i += 32) {
            key[i] = kInf;
            idx[i] = sentinel_of<IdxT>();
        }
    }

    // Threshold: the current k-th best (all lanes get the same value).
    __device__ __forceinline__ void threshold(float& tk, int64_t& ti) const {
        tk = key[k - 1];
        ti = static_cast<int64_t>(idx[k - 1]);
    }

    // Insert one candidate known to beat the threshold.  All 32 lanes call it
    // with the same (x, jx).  Cost ~ (k/32) x (2 loads + compare + ballot).
    __device__ void insert(float x, int64_t jx, int lane) {
        const int chunks = (k + 31) >> 5;
        int pos = 0;
        for (int r = 0; r < chunks; ++r) {
            const int i = lane + (r << 5);
            bool lt = false;
            if (i < k) lt = pair_less(key[i], static_cast<int64_t>(idx[i]), x, jx);
            pos += __popc(__ballot_sync(0xffffffffu, lt));
        }
        // shift [pos, k-1) up by one, high chunks first
        for (int r = chunks - 1; r >= 0; --r) {
            const int i = lane + (r << 5);
            if ((r << 5) + 31 < pos) break;  // whole chunk below pos: untouched (warp-uniform)
            float nk = 0.f;
            IdxT ni = 0;
            const bool mv = i < k && i > pos;
            if (mv) {
                nk = key[i - 1];
                ni = idx[i - 1];
            }
            __syncwarp();
            if (mv) {
                key[i] = nk;
                idx[i] = ni;
            } else if (i == pos) {
                key[i] = x;
                idx[i] = static_cast<IdxT>(jx);
            }
            __syncwarp();
        }
    }

    // Offer up to 32 x P candidates held P per lane (keys/indices in small
    // register arrays, invalid ones = +inf / sentinel).  Inserts every one that
    // beats the running threshold, in any order (the list is order-free).
    template <int P>
    __device__ void offer(const float (&ck)[P], const int64_t (&ci)[P], int lane) {
        float tk;
        int64_t ti;
        threshold(tk, ti);
        unsigned pending = 0;
#pragma unroll
        for (int p = 0; p < P; ++p)
            if (pair_less(ck[p], ci[p], tk, ti)) pending |= 1u << p;
        while (__any_sync(0xffffffffu, pending != 0)) {
            // each lane exposes its lowest pending candidate
            float myk = kInf;
            int64_t myi = kSentinelIdx;
            int myp = -1;
            if (pending) {
                myp = __ffs(pending) - 1;
#pragma unroll
                for (int p = 0; p < P; ++p)
                    if (p == myp) {
                        myk = ck[p];
                        myi = ci[p];
                    }
            }
            unsigned who = __ballot_sync(0xffffffffu, pending != 0);
            while (who) {
                const int src = __ffs(who) - 1;
                who &= who - 1;
                const float x = __shfl_sync(0xffffffffu, myk, src);
                const int64_t jx = __shfl_sync(0xffffffffu, myi, src);
                if (pair_less(x, jx, tk, ti)) {
                    insert(x, jx, lane);
                    threshold(tk, ti);
                }
            }
            if (myp >= 0) pending &= ~(1u << myp);
            // drop what the tightened threshold now rejects
#pragma unroll
            for (int p = 0; p < P; ++p)
                if ((pending >> p) & 1u)
                    if (!pair_less(ck[p], ci[p], tk, ti)) pending &= ~(1u << p);
        }
    }
};

// Register-resident variant for a burst of offers to one list with k <= 32 P:
// the list (same storage and order as WarpList) is loaded into registers,
// entry e = lane + 32 j in key[j] / idx[j], updated with warp shuffles (no
// shared-memory round trip per insertion) and written back once.
template <int P>
struct WarpRegList {
    float key[P];
    int32_t idx[P];

    __device__ __forceinline__ void load(const float* lk, const int32_t* li, int k, int lane) {
#pragma unroll
        for (int j = 0; j < P; ++j) {
            const int e = lane + 32 * j;
            key[j] = e < k ? lk[e] : kInf;
            idx[j] = e < k ? li[e] : 0x7fffffff;
        }
    }
    __device__ __forceinline__ void store(float* lk, int32_t* li, int k, int lane) const {
#pragma unroll
        for (int j = 0; j < P; ++j) {
            const int e = lane + 32 * j;
            if (e < k) {
                lk[e] = key[j];
                li[e] = idx[j];
            }
        }
    }
    // k-th entry (the running threshold), on every lane
    __device__ __forceinline__ void threshold(int k, float& tk, int32_t& ti) const {
        const int e = k - 1, j = e >> 5;
        float kk = key[0];
        int32_t ii = idx[0];
#pragma unroll
        for (int jj = 1; jj < P; ++jj)
            if (jj == j) {
                kk = key[jj];
                ii = idx[jj];
            }
        tk = __shfl_sync(0xffffffffu, kk, e & 31);
        ti = __shfl_sync(0xffffffffu, ii, e & 31);
    }
    // insert (x, jx) (same on all lanes), known to beat the threshold
    __device__ __forceinline__ void insert(float x, int32_t jx, int k, int lane) {
        int pos = 0;
#pragma unroll
        for (int j = 0; j < P; ++j) {
            const bool lt = lane + 32 * j < k && pair_less(key[j], idx[j], x, jx);
            pos += __popc(__ballot_sync(0xffffffffu, lt));
        }
        float pk[P];
        int32_t pi[P];
#pragma unroll
        for (int j = 0; j < P; ++j) {  // predecessor of entry e (entry e - 1), from the old values
            pk[j] = __shfl_up_sync(0xffffffffu, key[j], 1);
            pi[j] = __shfl_up_sync(0xffffffffu, idx[j], 1);
            if (j > 0) {
                const float ck = __shfl_sync(0xffffffffu, key[j - 1], 31);
                const int32_t cj = __shfl_sync(0xffffffffu, idx[j - 1], 31);
                if (lane == 0) {
                    pk[j] = ck;
                    pi[j] = cj;
                }
            }
        }
#pragma unroll
        for (int j = 0; j < P; ++j) {
            const int e = lane + 32 * j;
            if (e > pos) {
                key[j] = pk[j];
                idx[j] = pi[j];
            } else if (e == pos) {
                key[j] = x;
                idx[j] = jx;
            }
        }
    }
    // Offer up to 32 x C candidates held C per lane (invalid = +inf / INT32_MAX);
    // inserts every one that beats the running threshold.  Returns whether the
    // list changed.
    template <int C>
    __device__ bool offer(const float (&ck)[C], const int32_t (&ci)[C], int k, int lane) {
        float tk;
        int32_t ti;
        threshold(k, tk, ti);
        unsigned pending = 0;
#pragma unroll
        for (int p = 0; p < C; ++p)
            if (pair_less(ck[p], ci[p], tk, ti)) pending |= 1u << p;
        bool changed = false;
        while (__any_sync(0xffffffffu, pending != 0)) {
            float myk = kInf;
            int32_t myi = 0x7fffffff;
            int myp = -1;
            if (pending) {
                myp = __ffs(pending) - 1;
#pragma unroll
                for (int p = 0; p < C; ++p)
                    if (p == myp) {
                        myk = ck[p];
                        myi = ci[p];
                    }
            }
            unsigned who = __ballot_sync(0xffffffffu, pending != 0);
            while (who) {
                const int src = __ffs(who) - 1;
                who &= who - 1;
                const float x = __shfl_sync(0xffffffffu, myk, src);
                const int32_t jx = __shfl_sync(0xffffffffu, myi, src);
                if (pair_less(x, jx, tk, ti)) {
                    insert(x, jx, k, lane);
                    threshold(k, tk, ti);
                    changed = true;
                }
            }
            if (myp >= 0) pending &= ~(1u << myp);
#pragma unroll
            for (int p = 0; p < C; ++p)
                if ((pending >> p) & 1u)
                    if (!pair_less(ck[p], ci[p], tk, ti)) pending &= ~(1u << p);
        }
        return changed;
    }
};

// Finalize a sorted list in place (sqrt for L2) and restore the reference's
// table invariant (test_bruteforce.cpp:22-39: equal reported distances appear
// in ascending index order).  Two distinct squared keys can round to the same
// sqrtf, so after finalization a run of equal distances may hold indices out
// of order; keys were ascending, so runs are contiguous and short and one
// lane's insertion pass fixes them in O(k + inversions).
template <typename IdxT>
__device__ void finalize_list(float* key, IdxT* idx, int k, int metric, int lane) {
    for (int t = lane; t < k; t += 32) key[t] = finalize_key_rt(metric, key[t]);
    __syncwarp();
    if (metric == kL2 && lane == 0) {
        for (int t = 1; t < k; ++t) {
            const float v = key[t];
            const IdxT j = idx[t];
            int u = t;
            while (u > 0 && key[u - 1] == v && idx[u - 1] > j) {
                idx[u] = idx[u - 1];
                --u;
            }
            idx[u] = j;
        }
    }
    __syncwarp();
}

// finalize_list for L2 with the fix-up spread over the warp: keys were
// ascending, so after sqrt every run of equal distances is contiguous; the lane
// owning a run's first slot insertion-sorts the run's indices.
template <typename IdxT>
__device__ void finalize_list_runs(float* key, IdxT* idx, int k, int lane) {
    for (int t = lane; t < k; t += 32) key[t] = __fsqrt_rn(key[t]);
    __syncwarp();
    for (int t = lane; t < k; t += 32) {
        if (t > 0 && key[t - 1] == key[t]) continue;
        int e = t + 1;
        while (e < k && key[e] == key[t]) ++e;
        for (int x = t + 1; x < e; ++x) {
            const IdxT j = idx[x];
            int u = x;
            while (u > t && idx[u - 1] > j) {
                idx[u] = idx[u - 1];
                --u;
            }
            idx[u] = j;
        }
    }
    __syncwarp();
}

}  // namespace knnb200
