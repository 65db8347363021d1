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

// Large-k selection, one 256-thread block per query: gather the query's
// logged {A, index} values, bitonic-sort them by A, A_(k) = k-th; certify
// (>= k logged, no overflow, thresh(A_(k)) <= T0); exact FP32 keys of every
// value <= thresh(A_(k)); bitonic sort by (key, index); top k.
#ifndef KNN_DBG_LARGE
#define KNN_DBG_LARGE 0
#endif

// NT threads per query: the fewest of 64 / 128 / 256 / 512 that hold the candidate
// capacity NC <= 16 x NT (more resident blocks, cheaper barriers)
template <int NT>
__global__ void __launch_bounds__(NT, 65536 / (NT * 64)) select_large_kernel(LargeArgs a) {  // <= 64 registers
    sm100::pdl_wait();  // the fixed filter's logs are complete
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float* sk = reinterpret_cast<float*>(smem_raw);   // [NC]
    int* si = reinterpret_cast<int*>(sk + a.NC);       // [NC]
    __shared__ int s_off[33];
    __shared__ int s_cnt;
    __shared__ int s_sel[2];
    __shared__ unsigned s_hist[256];
    const int64_t q = blockIdx.x;
    const int qt = static_cast<int>(q / TILE), row = static_cast<int>(q % TILE);
    const int64_t p0 = static_cast<int64_t>(qt) * a.S_max;
    const int k = a.k;
    if (threadIdx.x == 0) {
        int off = 0;
        bool over = false;
        const int pair = qt >> 1;  // slots written: one per CTA touching the pair
        const int nslots = a.f.pair_slots[pair];
        for (int p = 0; p < a.S_max; ++p) {
            const int np = p < nslots ? a.f.log_n[(p0 + p) * TILE + row] : 0;
            over |= np > a.f.CV;
            s_off[p] = off;
            off += min(np, a.f.CV);
        }
        s_off[a.S_max] = off;
        s_cnt = over ? -1 : off;
    }
    __syncthreads();
    const int total = s_cnt;
    const float T0 = a.f.t0[q];
    bool ok = total >= k && total <= a.NC;
    float tau = kInf;
    int nc = 0;
    if (ok) {
        for (int p = 0; p < a.S_max; ++p) {
            const int o = s_off[p], np = s_off[p + 1] - o;
            const float2* src = a.f.vlog + ((p0 + p) * TILE + row) * a.f.CV;
            for (int e = threadIdx.x; e < np; e += blockDim.x) {
                const float2 r = src[e];
                sk[o + e] = r.x;
                si[o + e] = __float_as_int(r.y);
            }
        }
        __syncthreads();
        // a bound B >= A_(k) from one histogram pass (at most one of 256 bins
        // above A_(k): a few more candidates than thresh(A_(k)), all valid)
        const float ak = block_kth_upper_bound(sk, total, k, T0, s_hist, reinterpret_cast<unsigned*>(s_sel));
        const Consts qc = load_consts(a.f, q);
        tau = thresh(ak, qc);
        ok = tau <= T0;  // every reference with A <= tau was logged
        if (ok) {
            // compact the candidates (A <= tau) to the front in log order, i.e.
            // ascending reference index (parts in slot order, each part's log in
            // stream order); thread t owns the contiguous range [t per, t per + per)
            const int per = (total + NT - 1) / NT;  // <= NC / NT <= 16
            const int e0 = min(total, static_cast<int>(threadIdx.x) * per), e1 = min(total, e0 + per);
            int mine[16];
            int nm = 0;
            for (int e = e0; e < e1; ++e)
                if (sk[e] <= tau) mine[nm++] = si[e];
            const int base = block_exclusive_scan<NT>(nm, &nc);
            for (int j = 0; j < nm; ++j) si[base + j] = mine[j];
            __syncthreads();
        }
    }
    if (!ok) {
        if (threadIdx.x == 0) {
            const int slot = atomicAdd(a.fb_count, 1);
            a.fb_list[slot] = a.fb_offset + static_cast<int>(q);
            if (KNN_DBG_LARGE && slot < 8)
                printf("[select_large] q=%lld total=%d k=%d NC=%d tau=%g T0=%g nc=%d\n",
                       static_cast<long long>(q), total, k, a.NC, tau, T0, nc);
        }
        return;
    }
    // exact keys of the nc candidates (their indices are si[0..nc))
    const float* qrow = a.Q + q * a.d;
    for (int c = threadIdx.x; c < nc; c += blockDim.x)
        sk[c] = exact_key_l2(qrow, a.R + static_cast<int64_t>(si[c]) * a.d, a.d);
    // Preselection: when the candidates need a longer network than k does,
    // keep exactly the k smallest under the (key, index) order first -- every
    // key below the k-th smallest K, then the lowest-index entries equal to K
    // (the array is in ascending index order) -- so the bitonic network sorts
    // k rounded up to a power of two (k = 1024: 1024 instead of 2048 entries
    // for the ~1.1k candidates).
    int N2 = 32, Nk = 32;
    while (N2 < nc) N2 <<= 1;
    while (Nk < k) Nk <<= 1;
    __syncthreads();
    if (N2 > Nk) {
        const float K = block_kth_smallest(sk, nc, k, s_hist, s_sel);
        const int per = (nc + NT - 1) / NT;
        const int e0 = min(nc, static_cast<int>(threadIdx.x) * per), e1 = min(nc, e0 + per);
        int nl = 0, ne = 0;
        for (int e = e0; e < e1; ++e) {
            nl += sk[e] < K ? 1 : 0;
            ne += sk[e] == K ? 1 : 0;
        }
        int tot_less = 0, tot_eq = 0;
        block_exclusive_scan<NT>(nl, &tot_less);
        const int eq_before = block_exclusive_scan<NT>(ne, &tot_eq);
        const int need_eq = k - tot_less;  // >= 1 (K is the k-th smallest)
        float mk[16];
        int mi[16];
        int nm = 0, eq_seen = eq_before;
        for (int e = e0; e < e1; ++e) {
            const float x = sk[e];
            const bool keep = x < K || (x == K && eq_seen++ < need_eq);
            if (keep) {
                mk[nm] = x;
                mi[nm] = si[e];
                ++nm;
            }
        }
        int kept = 0;
        const int base = block_exclusive_scan<NT>(nm, &kept);  // kept == k
        for (int j = 0; j < nm; ++j) {
            sk[base + j] = mk[j];
            si[base + j] = mi[j];
        }
        nc = kept;
        N2 = Nk;
    }
    for (int e = nc + threadIdx.x; e < N2; e += blockDim.x) {
        sk[e] = kInf;
        si[e] = 0x7fffffff;
    }
    bitonic_sort_kv(sk, si, N2);
    // finalize: sqrt, then equal reported distances in ascending index order
    if (!a.raw_keys) {
        for (int t = threadIdx.x; t < k; t += blockDim.x) sk[t] = __fsqrt_rn(sk[t]);
        __syncthreads();
        // equal reported distances in ascending index order: each run of
        // equal distances (keys were ascending, so runs are contiguous and
        // short) is insertion-sorted by the thread owning its first slot
        for (int t = threadIdx.x; t < k; t += blockDim.x) {
            if (t > 0 && sk[t - 1] == sk[t]) continue;
            int e = t + 1;
            while (e < k && sk[e] == sk[t]) ++e;
            for (int x = t + 1; x < e; ++x) {
                const int j = si[x];
                int u = x;
                while (u > t && si[u - 1] > j) {
                    si[u] = si[u - 1];
                    --u;
                }
                si[u] = j;
            }
        }
        __syncthreads();
    }
    for (int t = threadIdx.x; t < k; t += blockDim.x) {
        a.out[q * k + t] = sk[t];
        a.out_idx[q * k + t] = a.index_base + si[t];
    }
}

}  // namespace

void launch_select_large(const LargeArgs& la, cudaStream_t stream) {
    const size_t smem = static_cast<size_t>(la.NC) * 8;
    const int NC = la.NC;
    const int nt = NC <= 16 * 64 ? 64 : NC <= 16 * 128 ? 128 : NC <= 16 * 256 ? 256 : LK_THREADS;
    auto sel = nt == 64    ? select_large_kernel<64>
               : nt == 128 ? select_large_kernel<128>
               : nt == 256 ? select_large_kernel<256> : select_large_kernel<LK_THREADS>;
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
