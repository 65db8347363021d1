// tensor_select.cu -- large-k selection (k > 32): one block per query
// certifies the fixed threshold, computes the exact FP32 keys of the values
// inside the bound and sorts them (register/shuffle bitonic network, block
// radix select).  DESIGN.md sec. 3.3.
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

using namespace sel;

// Large-k selection, one block per query.  The query's value logs (one per
// part slot, {A, index}) stay in global memory and are streamed (L1/L2 hits
// after the first pass); shared memory holds only the candidates:
//  1. a bound B >= A_(k): a 256-bin histogram over [-|q~|^2, T0], B = the upper
//     edge of the bin where the running count reaches k (at most one bin
//     above A_(k));
//  2. certificate: >= k values logged, no log overflowed, thresh(B) <= T0
//     (every reference with A <= tau = thresh(B) was logged);
//  3. candidates = logged values <= tau (warp-aggregated appends, at most NCC);
//  4. their exact FP32 keys; 5. the k smallest under the (key, index) order
//     by a bucket sort (block_bucket_topk), or a bitonic sort of all
//     candidates when the keys do not spread (dense ties).
// Candidate order is irrelevant: every comparison uses (key, index).
#ifndef KNN_DBG_LARGE
#define KNN_DBG_LARGE 0
#endif

template <int NT>
__global__ void __launch_bounds__(NT, 65536 / (NT * 64)) select_large_kernel(LargeArgs a) {  // <= 64 registers
    sm100::pdl_wait();  // the fixed filter's logs are complete
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int NCC = a.NC;                               // candidate capacity (power of two)
    const int k = a.k;
    float* sk = reinterpret_cast<float*>(smem_raw);    // [NCC] candidate keys
    int* si = reinterpret_cast<int*>(sk + NCC);         // [NCC] candidate indices
    float* ok = reinterpret_cast<float*>(si + NCC);     // [k + 32] bucket output keys
    int* oi = reinterpret_cast<int*>(ok + k + 32);      // [k + 32] bucket output indices
    unsigned* cnt = reinterpret_cast<unsigned*>(                 // [NCC] bucket counters, 16 B aligned
        (reinterpret_cast<uintptr_t>(oi + k + 32) + 15) & ~static_cast<uintptr_t>(15));
    __shared__ int s_np[32];
    __shared__ int s_total, s_nc, s_bin;
    __shared__ unsigned s_red[3];
    __shared__ unsigned s_hist[256];
    const int t = threadIdx.x, lane = t & 31;
    const int64_t q = blockIdx.x;
    const int qt = static_cast<int>(q / TILE), row = static_cast<int>(q % TILE);
    const int64_t p0 = static_cast<int64_t>(qt) * a.S_max;
    const int nparts = a.f.pair_slots[qt >> 1];  // slots written: one per CTA touching the pair
    for (int b = t; b < 256; b += NT) s_hist[b] = 0u;
    if (t < 32) {
        const int np = t < nparts ? a.f.log_n[(p0 + t) * TILE + row] : 0;
        const bool over = __any_sync(0xffffffffu, np > a.f.CV);
        const int c = min(np, a.f.CV);
        s_np[t] = c;
        const int tot = static_cast<int>(__reduce_add_sync(0xffffffffu, static_cast<unsigned>(c)));
        if (t == 0) {
            s_total = over ? -1 : tot;
            s_nc = 0;
            s_red[0] = 0xffffffffu;
            s_red[1] = 0u;
            s_red[2] = 0u;
        }
    }
    __syncthreads();
    const int total = s_total;
    const float T0 = a.f.t0[q];
    auto logp = [&](int p) { return a.f.vlog + ((p0 + p) * TILE + row) * a.f.CV; };
    // every logged value of the query (part by part), LU loads in flight per
    // thread before any is used: the passes are latency-bound otherwise
    // (one L2 round trip per NT values)
    constexpr int LU = 8;
    auto for_each_value = [&](auto&& fn) {
        for (int p = 0; p < nparts; ++p) {
            const float2* src = logp(p);
            const int np = s_np[p];
            for (int e0 = t; e0 < np; e0 += LU * NT) {
                float v[LU];
#pragma unroll
                for (int u = 0; u < LU; ++u) v[u] = e0 + u * NT < np ? __ldg(&src[e0 + u * NT].x) : kInf;
#pragma unroll
                for (int u = 0; u < LU; ++u) fn(v[u]);
            }
        }
    };
    bool ok_q = total >= k;
    float tau = kInf;
    int nc = 0;
    if (ok_q) {
        // 1. the bound.  256 bins over [lo, T0]: every logged value is <= T0,
        //    and A = D^2 - ||q~||^2 >= lo = -(||q~||^2 + eps) up to rounding
        //    (below lo -> bin 0).  Only when T0 is infinite (everything was
        //    logged, +inf padding included) a first pass finds the largest
        //    finite value.
        const Consts qc = load_consts(a.f, q);
        const float lo = -(qc.nq + qc.eps);
        float hi_f = T0;
        if (!(T0 < kInf)) {  // block-uniform
            unsigned hi_l = 0u;
            for_each_value([&](float v) {
                if (v < kInf) hi_l = max(hi_l, ord(v));
            });
            hi_l = __reduce_max_sync(0xffffffffu, hi_l);
            if (lane == 0) atomicMax(s_red + 1, hi_l);
            __syncthreads();
            hi_f = unord(s_red[1]);
        }
        const float scale = hi_f > lo && hi_f < kInf ? 256.f / (hi_f - lo) : 0.f;
        auto bin_of = [&](float v) { return min(255, max(0, static_cast<int>((v - lo) * scale))); };
        for_each_value([&](float v) {
            if (v < kInf) atomicAdd(s_hist + bin_of(v), 1u);
        });
        __syncthreads();
        if (t < 32) {  // warp 0: the bin where the running count reaches k
            unsigned c[8], tot = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                c[j] = s_hist[8 * t + j];
                tot += c[j];
            }
            unsigned incl = tot;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
                if (t >= o) incl += y;
            }
            const unsigned excl = incl - tot;
            if (t == 31 && incl < static_cast<unsigned>(k)) s_bin = -1;  // fewer than k finite values
            if (excl < static_cast<unsigned>(k) && static_cast<unsigned>(k) <= incl) {
                unsigned acc = excl;
                int j = 0;
                for (; j < 7; ++j) {
                    if (acc + c[j] >= static_cast<unsigned>(k)) break;
                    acc += c[j];
                }
                s_bin = 8 * t + j;
            }
        }
        __syncthreads();
        const int bk = s_bin;
        // B = the upper edge of bin bk: >= every value in the bins up to bk,
        // so >= A_(k) (the margin, 2^-18 of the larger magnitude, covers the
        // roundings of (v - lo) * scale and of the edge); the last bin's edge
        // is hi_f itself
        float B = kInf;
        if (bk >= 0)
            B = bk == 255 || !(scale > 0.f)
                    ? hi_f
                    : fminf(hi_f, lo + static_cast<float>(bk + 1) / scale +
                                      (fabsf(lo) + fabsf(hi_f)) * 0x1.0p-18f);
        // 2. certificate
        tau = bk >= 0 ? thresh(B, qc) : kInf;
        ok_q = tau <= T0;  // every reference with A <= tau was logged
        if (ok_q) {
            // 3. candidates: warp-aggregated appends (order is irrelevant)
            for (int p = 0; p < nparts; ++p) {
                const float2* src = logp(p);
                const int np = s_np[p];
                constexpr int CU = 4;
                for (int e0 = 0; e0 < np; e0 += CU * NT) {
                    float2 r[CU];
#pragma unroll
                    for (int u = 0; u < CU; ++u) {
                        const int e = e0 + u * NT + t;
                        r[u] = e < np ? __ldg(&src[e]) : make_float2(kInf, 0.f);
                    }
#pragma unroll
                    for (int u = 0; u < CU; ++u) {
                        const bool in = r[u].x <= tau;
                        const unsigned bal = __ballot_sync(0xffffffffu, in);
                        int base = 0;
                        if (lane == 0 && bal) base = atomicAdd(&s_nc, __popc(bal));
                        base = __shfl_sync(0xffffffffu, base, 0);
                        const int pos = base + __popc(bal & ((1u << lane) - 1u));
                        if (in && pos < NCC) si[pos] = __float_as_int(r[u].y);
                    }
                }
            }
            __syncthreads();
            nc = s_nc;
            ok_q = nc >= k && nc <= NCC;
        }
    }
    if (!ok_q) {
        if (t == 0) {
            const int slot = atomicAdd(a.fb_count, 1);
            a.fb_list[slot] = a.fb_offset + static_cast<int>(q);
            if (KNN_DBG_LARGE && slot < 8)
                printf("[select_large] q=%lld total=%d k=%d NCC=%d tau=%g T0=%g nc=%d\n",
                       static_cast<long long>(q), total, k, NCC, tau, T0, nc);
        }
        return;
    }
    // 4. exact keys of the nc candidates
    const float* qrow = a.Q + q * a.d;
    for (int c = t; c < nc; c += NT) sk[c] = exact_key_l2(qrow, a.R + static_cast<int64_t>(si[c]) * a.d, a.d);
    __syncthreads();
    // 5. the k smallest: bucket sort, or (dense ties) a bitonic sort of all
    int nbk = 32;
    while (nbk < nc) nbk <<= 1;
    float* rk = sk;
    int* ri = si;
    if (!block_bucket_topk<NT>(sk, si, nc, k, ok, oi, cnt, nbk, s_red)) {
        for (int e = nc + t; e < nbk; e += NT) {
            sk[e] = kInf;
            si[e] = 0x7fffffff;
        }
        bitonic_sort_kv(sk, si, nbk);
    }
    // finalize: sqrt, then equal reported distances in ascending index order
    if (!a.raw_keys) {
        for (int e = t; e < k; e += NT) rk[e] = __fsqrt_rn(rk[e]);
        __syncthreads();
        // each run of equal distances (keys were ascending, so runs are
        // contiguous and short) is insertion-sorted by the thread owning its
        // first slot
        for (int e = t; e < k; e += NT) {
            if (e > 0 && rk[e - 1] == rk[e]) continue;
            int f = e + 1;
            while (f < k && rk[f] == rk[e]) ++f;
            for (int x = e + 1; x < f; ++x) {
                const int j = ri[x];
                int u = x;
                while (u > e && ri[u - 1] > j) {
                    ri[u] = ri[u - 1];
                    --u;
                }
                ri[u] = j;
            }
        }
        __syncthreads();
    }
    for (int e = t; e < k; e += NT) {
        a.out[q * k + e] = rk[e];
        a.out_idx[q * k + e] = a.index_base + ri[e];
    }
}

}  // namespace

void launch_select_large(const LargeArgs& la, cudaStream_t stream) {
    // candidates [NC] keys + indices, bucket output [k + 32] x 2, counters [NC]
    const size_t smem = static_cast<size_t>(la.NC) * 12 + static_cast<size_t>(la.k + 32) * 8 + 16;
    // the fewest threads with <= 8 candidates each (<= 16 for the bitonic
    // fallback's register network)
    const int nt = la.NC <= 512 ? 64 : la.NC <= 1024 ? 128 : la.NC <= 2048 ? 256 : 512;
    auto sel = nt == 64    ? select_large_kernel<64>
               : nt == 128 ? select_large_kernel<128>
               : nt == 256 ? select_large_kernel<256> : select_large_kernel<512>;
    KNN_CUDA_CHECK(cudaFuncSetAttribute(sel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(smem)));
    {
        ProfileScope ps(stream, "select_large_kernel");
        KNN_CUDA_CHECK(launch_kernel(sel, static_cast<unsigned>(la.n), nt, smem, stream, pdl_enabled(2), la));
    }
    KNN_LAUNCH_CHECK();
}

}  // namespace tp
}  // namespace knnb200
