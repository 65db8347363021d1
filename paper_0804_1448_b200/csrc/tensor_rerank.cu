// tensor_rerank.cu -- the small-k exact re-rank (warp per query: bound from
// the union of the part lists, certificate, candidates from the group log,
// exact FP32 keys, exact top-k) and the gather / scatter of the host-driven
// fallback.  DESIGN.md sec. 3.2 step 3-4.
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdio>

#include "common.cuh"
#include "profile.cuh"
#include "sm100.cuh"
#include "tensor_internal.cuh"
#include "select_common.cuh"
#include "warp_list.cuh"

namespace knnb200 {
namespace tp {

namespace {

#ifndef KNN_RR_MERGE_MAX
#define KNN_RR_MERGE_MAX 16  // up to this many part lists: pairwise merges, more: bisection
#endif

// Warp per query.  (1) A_bound = k-th smallest of the union of the parts'
// bound lists (merge-path split over two lists, pairwise merges up to
// KNN_RR_MERGE_MAX lists, value bisection beyond); tau = thresh(A_bound).
// (2) Certificate: no part's group log overflowed, so every reference with
// A <= tau is in a log (every filter bound was >= tau).  (3) Candidates =
// logged values <= tau; their exact FP32 keys (key_step<kL2>, bitwise the
// exact kernel's arithmetic); (4) exact top-k by (key, index) rank counting.
__global__ void __launch_bounds__(RR_WARPS * 32) rerank_kernel(RerankArgs a) {
    sm100::pdl_wait();  // the filter's lists and logs are complete
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int64_t q = static_cast<int64_t>(blockIdx.x) * RR_WARPS + warp;
    if (q >= a.n) return;
    const int k = a.k;
    const int Kq = a.Kq;
    const int parts = a.S_max;  // <= 32 (checked on the host)
    const int span = parts * Kq;
    unsigned char* wb = smem_raw + static_cast<size_t>(warp) * rr_warp_bytes(span, k);
    float* sv = reinterpret_cast<float*>(wb);                 // [span] compacted bound lists
    float* ck = sv + span;                                     // [RR_CAND] exact keys
    int* ci = reinterpret_cast<int*>(ck + RR_CAND);            // [RR_CAND] reference indices
    float* fk = reinterpret_cast<float*>(ci + RR_CAND);        // [k] result keys
    int64_t* fi = reinterpret_cast<int64_t*>(
        wb + ((static_cast<size_t>(span) * 4 + RR_CAND * 8 + static_cast<size_t>(k) * 4 + 15) / 16) * 16);
    int* gcol = reinterpret_cast<int*>(fi + k);                // [RR_CAND] first column of in-tau groups

    const int qt = static_cast<int>(q / TILE);
    const int row = static_cast<int>(q % TILE);
    const int64_t p0 = static_cast<int64_t>(qt) * parts;

    // Every step below issues its loads for the whole query at once (one
    // memory round trip per step): the kernel is latency-bound per warp.
    // part slots written for this pair: one per CTA whose unit range touches it
    const int pair = qt >> 1;
    const int nslots = a.f.pair_slots[pair];
    // Counts and the first two lists are read speculatively for every part
    // slot of the tile (in bounds; slots >= nslots and entries past cnt are
    // stale and masked), in the same memory round trip as nslots.
    int cnt = 0, nlog = 0;
    if (lane < parts) {
        cnt = a.f.part_cnt[(p0 + lane) * TILE + row];
        nlog = a.f.log_n[(p0 + lane) * TILE + row];
    }
    float pa[2];
#pragma unroll
    for (int p = 0; p < 2; ++p)
        pa[p] = (p < parts && lane < Kq) ? a.f.part_A[((p0 + p) * TILE + row) * Kq + lane] : kInf;
    if (lane >= nslots) cnt = nlog = 0;
    const Consts qc = load_consts(a.f, q);
    // 0. all bound lists, compacted: list p's entries go to [excl_p, excl_p + cnt_p)
    int cincl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, cincl, o);
        if (lane >= o) cincl += y;
    }
    const int L = __shfl_sync(0xffffffffu, cincl, 31);
    if (nslots <= 2) {
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            const int cp = __shfl_sync(0xffffffffu, cnt, p);
            const int ep = __shfl_sync(0xffffffffu, cincl, p) - cp;
            if (p < nslots && lane < cp) sv[ep + lane] = pa[p];
        }
    } else {
        // many parts (short stream-K parts: small query sets, long reference
        // sets): 8 lists' loads in flight per round trip, not one
        for (int pb = 2; pb < nslots; pb += 8) {
            float v8[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int p = pb + u;
                const int cp = __shfl_sync(0xffffffffu, cnt, p & 31);
                v8[u] = (p < nslots && lane < cp) ? a.f.part_A[((p0 + p) * TILE + row) * Kq + lane] : kInf;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int p = pb + u;
                const int cp = __shfl_sync(0xffffffffu, cnt, p & 31);
                const int ep = __shfl_sync(0xffffffffu, cincl, p & 31) - cp;
                if (p < nslots && lane < cp) sv[ep + lane] = v8[u];
            }
        }
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            const int cp = __shfl_sync(0xffffffffu, cnt, p);
            const int ep = __shfl_sync(0xffffffffu, cincl, p) - cp;
            if (lane < cp) sv[ep + lane] = pa[p];
        }
    }
    __syncwarp();

    // 1. k-th smallest (value, position) of the compacted lists.  Each list is
    //    sorted, so an entry's rank is its own position plus, per other list,
    //    a binary search: entries <= v of earlier lists, < v of later ones.
    float B = kInf;
    if (L >= k && nslots <= 2) {
        // One or two lists (the common stream-K case): lane i tests the split
        // "i smallest of list 0, k-i of list 1"; every valid split takes a
        // multiset of the k smallest values, so its maximum is the k-th value.
        const int cA = __shfl_sync(0xffffffffu, cnt, 0);
        const int cB = L - cA;
        const float* sb = sv + cA;
        for (int i = lane; i <= k; i += 32) {
            const int j = k - i;
            if (i <= cA && j <= cB &&
                (i == 0 || j == cB || sv[i - 1] <= sb[j]) &&
                (j == 0 || i == cA || sb[j - 1] <= sv[i]))
                B = fmaxf(i > 0 ? sv[i - 1] : -kInf, j > 0 ? sb[j - 1] : -kInf);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) B = fminf(B, __shfl_xor_sync(0xffffffffu, B, o));
    } else if (L >= k && nslots <= KNN_RR_MERGE_MAX) {
        // A few lists: merge them one at a time, keeping the k smallest (lane t
        // places output t by a merge-path binary search); B = the k-th.
        const float* A = sv;
        int na = min(k, __shfl_sync(0xffffffffu, cnt, 0));
        float* dst = ck;
        for (int p = 1; p < nslots; ++p) {
            const int nb = __shfl_sync(0xffffffffu, cnt, p);
            const float* Bl = sv + __shfl_sync(0xffffffffu, cincl, p) - nb;
            const int out = min(k, na + nb);
            if (lane < out) {
                const int t = lane;
                int lo = max(0, t - nb), hi = min(t, na);  // A entries among the first t outputs
                while (lo < hi) {
                    const int md = (lo + hi) >> 1;
                    if (A[md] <= Bl[t - 1 - md]) lo = md + 1;
                    else hi = md;
                }
                const int j = t - lo;
                dst[t] = (lo < na && (j >= nb || A[lo] <= Bl[j])) ? A[lo] : Bl[j];
            }
            __syncwarp();
            A = dst;
            na = out;
            dst = dst == ck ? ck + 32 : ck;
        }
        B = A[k - 1];
    } else if (L >= k) {
        // More lists: bisection on the value.  Lane p counts the entries <= v
        // of its sorted list (binary search), the warp sums; the smallest v
        // (in float order) with count >= k is the k-th smallest entry.
        const int cp = lane < nslots ? cnt : 0;
        const int ep = cincl - cnt;
        unsigned lo = cp > 0 ? sel::ord(sv[ep]) : 0xffffffffu;
        unsigned hi = cp > 0 ? sel::ord(sv[ep + cp - 1]) : 0u;
        lo = __reduce_min_sync(0xffffffffu, lo);
        hi = __reduce_max_sync(0xffffffffu, hi);
        while (lo < hi) {  // warp-uniform
            const unsigned mid = lo + ((hi - lo) >> 1);
            const float v = sel::unord(mid);
            int a0 = 0, a1 = cp;  // entries of list `lane` that are <= v
            while (a0 < a1) {
                const int md = (a0 + a1) >> 1;
                if (sv[ep + md] <= v) a0 = md + 1;
                else a1 = md;
            }
            const int c = static_cast<int>(__reduce_add_sync(0xffffffffu, static_cast<unsigned>(a0)));
            if (c >= k) hi = mid;
            else lo = mid + 1;
        }
        B = sel::unord(lo);
    }
    const float tau = thresh(B, qc);

    // 2. certificate
    bool ok = __all_sync(0xffffffffu, nlog <= a.f.CG) && isfinite(tau);

    // 3. candidates: logged values <= tau.  Heads of every logged group of
    //    every part (flattened over parts), then the values of the groups whose
    //    minimum is inside tau, then their values <= tau.
    int nc = 0;
    auto head_of = [&](int64_t slot) { return reinterpret_cast<const int*>(a.f.log_h + slot); };
    auto log_slot = [&](int h) -> int64_t {
        return ((p0 + (h >> 16)) * TILE + row) * static_cast<int64_t>(a.f.CG) + (h & 0xffff);
    };
    if (ok) {
        int* gl = reinterpret_cast<int*>(ck);  // in-tau groups (part-relative handles), reuses ck
        const uint64_t pol = l2_evict_first_policy();  // the logs are read once
        int ng = 0;
        // log heads flattened over the parts (part-major), 8 per lane per
        // round so that one round trip covers up to 256 logged groups
        int nincl = nlog;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, nincl, o);
            if (lane >= o) nincl += y;
        }
        const int NT = __shfl_sync(0xffffffffu, nincl, 31);
        int* pend = reinterpret_cast<int*>(sv);  // part ends; the bound lists are consumed
        __syncwarp();
        if (lane < nslots) pend[lane] = nincl;
        __syncwarp();
        for (int t0 = 0; t0 < NT; t0 += 256) {
            float hv[8];
            int hs[8], hc[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const int t = t0 + e * 32 + lane;
                hv[e] = kInf;
                hs[e] = 0;
                hc[e] = 0;
                if (t < NT) {
                    // part of flat head t: the first part whose end exceeds t
                    int p = 0, b1 = nslots - 1;
                    while (p < b1) {
                        const int md = (p + b1) >> 1;
                        if (pend[md] <= t) p = md + 1;
                        else b1 = md;
                    }
                    const int ex = p > 0 ? pend[p - 1] : 0;
                    // part-relative handle (part << 16 | slot, CG <= 4096): the global
                    // slot needs 64 bits once parts * 128 * CG >= 2^31
                    hs[e] = (p << 16) | (t - ex);
                    // the whole head {minimum, first column}: the column of an
                    // in-tau group is then at hand for the value step
                    const int2 h2 = ldg2_hint(head_of(log_slot(hs[e])), pol);
                    hv[e] = __int_as_float(h2.x);
                    hc[e] = h2.y;
                }
            }
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const bool in = hv[e] <= tau;
                const unsigned bal = __ballot_sync(0xffffffffu, in);
                const int pos = ng + __popc(bal & ((1u << lane) - 1u));
                if (in && pos < RR_CAND) {
                    gl[pos] = hs[e];
                    gcol[pos] = hc[e];
                }
                ng += __popc(bal);
            }
        }
        ok = ng <= RR_CAND;
        __syncwarp();
        for (int j0 = 0; ok && j0 < ng; j0 += 32) {
            const int j = j0 + lane;
            float w[8];
            int c0 = 0;
#pragma unroll
            for (int e = 0; e < 8; ++e) w[e] = kInf;
            if (j < ng) {
                const int64_t slot = log_slot(gl[j]);
                ldg8_hint(reinterpret_cast<const float*>(a.f.log_v + 2 * slot), w, pol);
                c0 = gcol[j];
            }
            __syncwarp();
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const bool c = w[e] <= tau;
                const unsigned bal = __ballot_sync(0xffffffffu, c);
                const int pos = nc + __popc(bal & ((1u << lane) - 1u));
                if (c && pos < RR_CAND) ci[pos] = c0 + e;
                nc += __popc(bal);
            }
        }
        ok = ok && nc <= RR_CAND && nc >= k;  // heavy ties beyond the fast path: exact kernel
        if (kStats && a.f.stats && ok && lane == 0) {
            atomicAdd(a.f.stats + 0, static_cast<unsigned long long>(nc));
            atomicAdd(a.f.stats + 1, static_cast<unsigned long long>(ng));
            atomicAdd(a.f.stats + 2, 1ull);
            atomicAdd(a.f.stats + 3, static_cast<unsigned long long>(NT));
            atomicAdd(a.f.stats + 4, static_cast<unsigned long long>(nslots));
        }
    }
    if (!ok) {
        if (lane == 0) {
            const int slot = atomicAdd(a.fb_count, 1);
            a.fb_list[slot] = a.fb_offset + static_cast<int>(q);
        }
        return;
    }
    __syncwarp();

    // 4. exact FP32 keys of the candidates (lane-parallel, fixed coordinate order)
    const float* qrow = a.Q + q * a.d;
    for (int c = lane; c < nc; c += 32)
        ck[c] = exact_key_l2(qrow, a.R + static_cast<int64_t>(ci[c]) * a.d, a.d);
    __syncwarp();

    // 5. exact top-k under the (key, index) order: up to 32 candidates, one
    //    per lane, by a shuffle bitonic network; more, by rank counting
    if (nc <= 32) {
        float kc = lane < nc ? ck[lane] : kInf;
        int jc = lane < nc ? ci[lane] : 0x7fffffff;
#pragma unroll
        for (int size = 2; size <= 32; size <<= 1)
#pragma unroll
            for (int stride = size >> 1; stride > 0; stride >>= 1) {
                const float pk = __shfl_xor_sync(0xffffffffu, kc, stride);
                const int pj = __shfl_xor_sync(0xffffffffu, jc, stride);
                const bool keep_min = ((lane & stride) == 0) == ((lane & size) == 0);
                if (pair_less(pk, pj, kc, jc) == keep_min) {
                    kc = pk;
                    jc = pj;
                }
            }
        if (lane < k) {
            fk[lane] = kc;
            fi[lane] = jc;
        }
    } else {
        for (int c = lane; c < nc; c += 32) {
            const float kc = ck[c];
            const int jc = ci[c];
            int r = 0;
            for (int c2 = 0; c2 < nc; ++c2) r += pair_less(ck[c2], ci[c2], kc, jc) ? 1 : 0;
            if (r < k) {
                fk[r] = kc;
                fi[r] = jc;
            }
        }
    }
    __syncwarp();
    if (!a.raw_keys) finalize_list_runs(fk, fi, k, lane);
    for (int t = lane; t < k; t += 32) {
        a.out[q * k + t] = fk[t];
        a.out_idx[q * k + t] = a.index_base + fi[t];
    }
}

}  // namespace

void launch_rerank(const RerankArgs& ra, size_t smem, cudaStream_t stream) {
    {
        ProfileScope ps(stream, "rerank_kernel");
        KNN_CUDA_CHECK(launch_kernel(rerank_kernel,
                                     static_cast<unsigned>((ra.n + RR_WARPS - 1) / RR_WARPS),
                                     RR_WARPS * 32, smem, stream, pdl_enabled(2), ra));
    }
    KNN_LAUNCH_CHECK();
}

}  // namespace tp
}  // namespace knnb200
