// exact_large.cu -- large k (256 < k <= 1024) on the exact SIMT path (every
// metric; L2 lands here when the tensor path does not apply, e.g. d > 128).
//
// The reference keeps each query's k smallest keys (src/topk.cpp:17-33, heap
// select over the chunk's key row, bruteforce.cpp:81-96).  A running list of
// k in the hundreds does not fit registers or shared memory per query, and the
// global-memory list it used to need is ~100x slower than the key arithmetic.
// Instead, a fixed per-query threshold makes the selection a filter:
//   1. sample   exact keys of every query against a strided sample of
//               s = 32 m / (3 k) references (exact kernel, k' = 32, raw keys);
//               T0 = the 32nd smallest estimates the (3k)-th smallest key.
//   2. log      the exact kernel in threshold-log mode appends every key <= T0
//               (exact FP32, bitwise the list path's) with its index to a
//               per-(query, segment) log, in reference order.
//   3. select   block per query: A_(k) = k-th smallest logged key (radix
//               select), certified iff no log overflowed, >= k were logged and
//               A_(k) <= T0 (every key <= A_(k) is then in a log); keep the keys
//               below A_(k) and the lowest-index ties at A_(k) (the logs are in
//               ascending index order), sort them by (key, index), finalize.
//   4. fallback uncertified queries (a tail estimate of T0) run the list path.
// Results are bitwise the list path's: same keys, same (key, index) order.
#include <algorithm>
#include <cstdio>

#include "common.cuh"
#include "engine.cuh"
#include "exact_kernel.cuh"
#include "profile.cuh"
#include "select_common.cuh"
#include "sm100.cuh"
#include "warp_list.cuh"

namespace knnb200 {

namespace {

using namespace sel;

constexpr int kSeedRank = 32;   // T0 = the 32nd smallest sample key
constexpr int kMargin = 3;      // ... estimating the (3k)-th smallest key

// rows r * stride (r < s) of X into a contiguous s x d buffer
__global__ void gather_strided_kernel(const float* X, int d, int64_t stride, int64_t s, float* out) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= s * d) return;
    const int64_t r = i / d;
    out[i] = X[r * stride * d + (i - r * d)];
}

struct SelArgs {
    const float2* vlog;
    const int* vlog_n;
    int CV, NC, k;
    int64_t n;
    int ntiles, max_ctas;
    const float* t0;
    int t0_stride;
    int metric, raw_keys;
    int64_t index_base;
    float* out;
    int64_t* out_idx;
    int* fb_count;
    int* fb_list;
};

template <int NT>
__global__ void __launch_bounds__(NT) select_exact_kernel(SelArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float* sk = reinterpret_cast<float*>(smem_raw);  // [NC]
    int* si = reinterpret_cast<int*>(sk + a.NC);      // [NC]
    __shared__ int s_off[64];
    __shared__ int s_tot;
    __shared__ int s_sel[2];
    __shared__ unsigned s_hist[256];
    const int64_t q = blockIdx.x;
    const int64_t b = q / 128;
    const int row = static_cast<int>(q - b * 128);
    const int k = a.k;
    const ExactSplit sp = exact_split(a.n, a.ntiles, a.max_ctas);
    const int64_t first = sp.cta_of(b * a.ntiles), last = sp.cta_of((b + 1) * a.ntiles - 1);
    const int nparts = static_cast<int>(last - first + 1);
    auto part_base = [&](int p) { return (static_cast<size_t>(first + p + b) * 128 + row); };
    if (threadIdx.x == 0) {
        int off = 0;
        bool over = nparts > 63;
        for (int p = 0; p < nparts && !over; ++p) {
            const int np = a.vlog_n[part_base(p)];
            over |= np > a.CV;
            s_off[p] = off;
            off += min(np, a.CV);
        }
        s_off[min(nparts, 63)] = off;
        s_tot = over || off > a.NC ? -1 : off;
    }
    __syncthreads();
    const int total = s_tot;
    const float T0 = a.t0[q * a.t0_stride];
    bool ok = total >= k;
    float K = kInf;
    if (ok) {
        for (int p = 0; p < nparts; ++p) {  // logs in part (= reference) order
            const int o = s_off[p], np = s_off[p + 1] - o;
            const float2* src = a.vlog + part_base(p) * a.CV;
            for (int e = threadIdx.x; e < np; e += NT) {
                const float2 r = src[e];
                sk[o + e] = r.x;
                si[o + e] = __float_as_int(r.y);
            }
        }
        __syncthreads();
        K = block_kth_smallest(sk, total, k, s_hist, s_sel);
        ok = K <= T0;  // every key <= K was logged
    }
    if (!ok) {
        if (threadIdx.x == 0) {
            const int slot = atomicAdd(a.fb_count, 1);
            a.fb_list[slot] = static_cast<int>(q);
        }
        return;
    }
    // keep the k smallest under (key, index): keys < K, then the lowest-index
    // keys == K (the array is in ascending index order); thread t owns the
    // contiguous range [t per, t per + per)
    const int per = (total + NT - 1) / NT;  // <= NC / NT <= 16
    const int e0 = min(total, static_cast<int>(threadIdx.x) * per), e1 = min(total, e0 + per);
    int nl = 0, ne = 0;
    for (int e = e0; e < e1; ++e) {
        nl += sk[e] < K ? 1 : 0;
        ne += sk[e] == K ? 1 : 0;
    }
    int tot_less = 0, tot_eq = 0;
    block_exclusive_scan<NT>(nl, &tot_less);
    const int eq_before = block_exclusive_scan<NT>(ne, &tot_eq);
    const int need_eq = k - tot_less;
    float mk[16];
    int mi[16];
    int nm = 0, eq_seen = eq_before;
    for (int e = e0; e < e1; ++e) {
        const float x = sk[e];
        if (x < K || (x == K && eq_seen++ < need_eq)) {
            mk[nm] = x;
            mi[nm] = si[e];
            ++nm;
        }
    }
    int kept = 0;
    const int base = block_exclusive_scan<NT>(nm, &kept);
    for (int j = 0; j < nm; ++j) {
        sk[base + j] = mk[j];
        si[base + j] = mi[j];
    }
    int N2 = 32;
    while (N2 < k) N2 <<= 1;
    for (int e = k + threadIdx.x; e < N2; e += NT) {
        sk[e] = kInf;
        si[e] = 0x7fffffff;
    }
    bitonic_sort_kv(sk, si, N2);
    if (!a.raw_keys) {
        for (int t = threadIdx.x; t < k; t += NT) sk[t] = finalize_key_rt(a.metric, sk[t]);
        __syncthreads();
        if (a.metric == kL2) {  // equal reported distances in ascending index order
            for (int t = threadIdx.x; t < k; t += NT) {
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
    }
    for (int t = threadIdx.x; t < k; t += NT) {
        a.out[q * k + t] = sk[t];
        a.out_idx[q * k + t] = a.index_base + si[t];
    }
}

// gather / scatter of the fallback queries
__global__ void gather_list_kernel(const float* X, int d, const int* list, int count, float* out) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= static_cast<int64_t>(count) * d) return;
    const int64_t r = i / d;
    out[i] = X[static_cast<int64_t>(list[r]) * d + (i - r * d)];
}

__global__ void scatter_list_kernel(const float* sd, const int64_t* si, const int* list, int count, int k,
                                    float* out, int64_t* out_idx) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= static_cast<int64_t>(count) * k) return;
    const int64_t r = i / k;
    const int64_t dst = static_cast<int64_t>(list[r]) * k + (i - r * k);
    out[dst] = sd[i];
    out_idx[dst] = si[i];
}

}  // namespace

bool exact_large_applies(int64_t m, int k) {
    return k > static_cast<int>(exact_smem_list_limit_k()) && k <= 1024 && m >= 4096;
}

void run_exact_large(DeviceContext& ctx, cudaStream_t stream, const float* dQ, int64_t n,
                     const float* dR, int64_t m, int d, int k, int metric, int raw_keys,
                     int64_t index_base, float* d_out, int64_t* d_idx) {
    // 1. sample: every stride-th reference, s ~ kSeedRank m / (kMargin k) rows
    const int64_t stride = std::max<int64_t>(1, (static_cast<int64_t>(kMargin) * k) / kSeedRank);
    const int64_t s = (m + stride - 1) / stride;
    // 2. log pass scratch: per (segment slot, row) logs of CV entries
    const int ntiles = exact_ntiles(m);
    const int max_ctas = kSmCount * 2;
    const int64_t slots = exact_slots(n, ntiles, max_ctas);
    const int CV = 2 * kMargin * k + 256;
    int NC = 1;
    while (NC < 2 * kMargin * k) NC <<= 1;
    NC = std::min(NC, 16 * 512);
    Sizer sz;
    sz.take<float>(static_cast<size_t>(s) * d);
    sz.take<float>(static_cast<size_t>(n) * kSeedRank);
    sz.take<int64_t>(static_cast<size_t>(n) * kSeedRank);
    sz.take<float2>(static_cast<size_t>(slots) * 128 * CV);
    sz.take<int>(static_cast<size_t>(slots) * 128);
    sz.take<int>(static_cast<size_t>(n) + 1);
    const size_t own = sz.used + 256;
    // the sample search carves the context arena, so this path's buffers come
    // from a separate allocation (stream-ordered)
    char* mem = nullptr;
    KNN_CUDA_CHECK(cudaMallocAsync(reinterpret_cast<void**>(&mem), own, stream));
    Carver cv{mem};
    float* Rs = cv.take<float>(static_cast<size_t>(s) * d);
    float* sk32 = cv.take<float>(static_cast<size_t>(n) * kSeedRank);
    int64_t* si32 = cv.take<int64_t>(static_cast<size_t>(n) * kSeedRank);
    float2* vlog = cv.take<float2>(static_cast<size_t>(slots) * 128 * CV);
    int* vlog_n = cv.take<int>(static_cast<size_t>(slots) * 128);
    int* fb = cv.take<int>(static_cast<size_t>(n) + 1);
    {
        ProfileScope ps(stream, "exact_large_sample");
        const int64_t tot = s * d;
        gather_strided_kernel<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, stream>>>(dR, d, stride, s, Rs);
        KNN_LAUNCH_CHECK();
    }
    search_device(ctx, stream, dQ, n, Rs, s, d, std::min<int64_t>(kSeedRank, s) == kSeedRank ? kSeedRank : static_cast<int>(s),
                  metric, /*path=*/1, /*raw_keys=*/1, 0, sk32, si32, nullptr);
    // 2. the threshold-log pass
    ExactArgs a{};
    a.Q = dQ;
    a.R = dR;
    a.n = n;
    a.m = m;
    a.d = d;
    a.k = k;
    a.ntiles = ntiles;
    a.t0 = sk32 + (kSeedRank - 1);
    a.t0_stride = kSeedRank;
    a.vlog = vlog;
    a.vlog_n = vlog_n;
    a.CV = CV;
    launch_exact_log(metric, a, stream);
    // 3. select
    KNN_CUDA_CHECK(cudaMemsetAsync(fb, 0, sizeof(int), stream));
    SelArgs sa{};
    sa.vlog = vlog;
    sa.vlog_n = vlog_n;
    sa.CV = CV;
    sa.NC = NC;
    sa.k = k;
    sa.n = n;
    sa.ntiles = ntiles;
    sa.max_ctas = max_ctas;
    sa.t0 = a.t0;
    sa.t0_stride = kSeedRank;
    sa.metric = metric;
    sa.raw_keys = raw_keys;
    sa.index_base = index_base;
    sa.out = d_out;
    sa.out_idx = d_idx;
    sa.fb_count = fb;
    sa.fb_list = fb + 1;
    {
        const int nt = NC <= 16 * 256 ? 256 : 512;
        const size_t smem = static_cast<size_t>(NC) * 8;
        auto kern = nt == 256 ? select_exact_kernel<256> : select_exact_kernel<512>;
        KNN_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            static_cast<int>(smem)));
        ProfileScope ps(stream, "select_exact_kernel");
        kern<<<static_cast<unsigned>(n), nt, smem, stream>>>(sa);
        KNN_LAUNCH_CHECK();
    }
    // 4. uncertified queries: the list path (host-driven, rare)
    int fails = 0;
    KNN_CUDA_CHECK(cudaMemcpyAsync(&fails, fb, sizeof(int), cudaMemcpyDeviceToHost, stream));
    KNN_CUDA_CHECK(cudaStreamSynchronize(stream));
    if (fails > 0) {
        float* gq = nullptr;
        float* od = nullptr;
        int64_t* oi = nullptr;
        KNN_CUDA_CHECK(cudaMallocAsync(&gq, sizeof(float) * fails * d, stream));
        KNN_CUDA_CHECK(cudaMallocAsync(&od, sizeof(float) * fails * k, stream));
        KNN_CUDA_CHECK(cudaMallocAsync(&oi, sizeof(int64_t) * fails * k, stream));
        const int64_t tq = static_cast<int64_t>(fails) * d, to = static_cast<int64_t>(fails) * k;
        gather_list_kernel<<<static_cast<unsigned>((tq + 255) / 256), 256, 0, stream>>>(dQ, d, fb + 1, fails, gq);
        KNN_LAUNCH_CHECK();
        run_exact_lists(ctx, stream, gq, fails, dR, m, d, k, metric, raw_keys, index_base, od, oi);
        scatter_list_kernel<<<static_cast<unsigned>((to + 255) / 256), 256, 0, stream>>>(od, oi, fb + 1, fails, k,
                                                                                       d_out, d_idx);
        KNN_LAUNCH_CHECK();
        KNN_CUDA_CHECK(cudaFreeAsync(gq, stream));
        KNN_CUDA_CHECK(cudaFreeAsync(od, stream));
        KNN_CUDA_CHECK(cudaFreeAsync(oi, stream));
    }
    ctx.s->last_fallbacks = fails;
    KNN_CUDA_CHECK(cudaFreeAsync(mem, stream));
}

}  // namespace knnb200
