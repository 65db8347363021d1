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
//   4. fallback uncertified queries (a tail estimate of T0) run the list path
//               over a device-side row list.
// All of it is stream-ordered device work (no host round trip), and the same
// sequence serves a device-side query list (the tensor path's large-k
// certification fallback).
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
    const int* qlist;   // nullable: position i of the search is Q row / output row qlist[i]
    const int* qcount;  // nullable: device-side count of positions (<= n)
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
    const int64_t n_eff = a.qcount ? min(a.n, static_cast<int64_t>(*a.qcount)) : a.n;
    // block-stride over positions: a device-side count launches a fixed grid
    for (int64_t q = blockIdx.x; q < n_eff; q += gridDim.x) {  // position (logs are by position)
    __syncthreads();  // the previous position's shared-memory reads are done
    const int64_t orow = a.qlist ? static_cast<int64_t>(a.qlist[q]) : q;  // Q / output row
    const int64_t b = q / 128;
    const int row = static_cast<int>(q - b * 128);
    const int k = a.k;
    const ExactSplit sp = exact_split(n_eff, a.ntiles, a.max_ctas);
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
    const float T0 = a.t0[orow * a.t0_stride];
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
            a.fb_list[slot] = static_cast<int>(orow);
        }
        continue;
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
        a.out[orow * k + t] = sk[t];
        a.out_idx[orow * k + t] = a.index_base + si[t];
    }
    }
}

}  // namespace

bool exact_large_applies(int64_t m, int k) {
    return k > static_cast<int>(exact_smem_list_limit_k()) && k <= 1024 && m >= 4096;
}

namespace {
__global__ void add_count_kernel(int* acc, const int* src, bool first) {
    if (threadIdx.x == 0) *acc = (first ? 0 : *acc) + *src;
}
}  // namespace

static void run_exact_large_chunk(DeviceContext& ctx, cudaStream_t stream, const float* dQ, int64_t n,
                                  const float* dR, int64_t m, int d, int k, int metric, int raw_keys,
                                  int64_t index_base, float* d_out, int64_t* d_idx, const int* qlist,
                                  const int* qcount, int* fb_total, bool first);

// A host-known query set is processed in chunks of at most kChunk queries: the
// logs take (G + n / 128) x 128 x CV entries, so chunking bounds the scratch
// (k = 1024: ~3.6 GB per chunk).  A device-side list is one chunk (the tensor
// path's fallback list; its capacity is the search's own query count).
constexpr int64_t kChunk = 32768;

void run_exact_large(DeviceContext& ctx, cudaStream_t stream, const float* dQ, int64_t n,
                     const float* dR, int64_t m, int d, int k, int metric, int raw_keys,
                     int64_t index_base, float* d_out, int64_t* d_idx, const int* qlist,
                     const int* qcount) {
    if (qlist || n <= kChunk) {
        run_exact_large_chunk(ctx, stream, dQ, n, dR, m, d, k, metric, raw_keys, index_base, d_out, d_idx,
                              qlist, qcount, nullptr, true);
        return;
    }
    int* total = ctx.s->fb_dev;  // the fallback count over all chunks
    for (int64_t q0 = 0; q0 < n; q0 += kChunk) {
        const int64_t nq = std::min(kChunk, n - q0);
        run_exact_large_chunk(ctx, stream, dQ + q0 * d, nq, dR, m, d, k, metric, raw_keys, index_base,
                              d_out + q0 * k, d_idx + q0 * k, nullptr, nullptr, total, q0 == 0);
    }
    ctx.s->fb_on_device = total != nullptr;
}

static void run_exact_large_chunk(DeviceContext& ctx, cudaStream_t stream, const float* dQ, int64_t n,
                                  const float* dR, int64_t m, int d, int k, int metric, int raw_keys,
                                  int64_t index_base, float* d_out, int64_t* d_idx, const int* qlist,
                                  const int* qcount, int* fb_total, bool first) {
    // Everything below is stream-ordered device work: no host round trip, so
    // the search is asynchronous and graph-capturable; with (qlist, qcount)
    // it serves a device-side query list (the tensor path's certification
    // fallback).  Outputs and thresholds are indexed by the query's row,
    // logs by its position.
    // 1. sample: every stride-th reference, s ~ kSeedRank m / (kMargin k) rows
    const int64_t stride = std::max<int64_t>(1, (static_cast<int64_t>(kMargin) * k) / kSeedRank);
    const int64_t s = (m + stride - 1) / stride;
    const int ntiles = exact_ntiles(m), stiles = exact_ntiles(s);
    const int smax = exact_max_ctas(kSeedRank, true);
    const int lmax = exact_log_max_ctas();
    const int gmax = exact_max_ctas(k, false);
    const int64_t s_slots = exact_slots(n, stiles, smax);
    const int64_t l_slots = exact_slots(n, ntiles, lmax);
    const int64_t f_slots = exact_slots(n, ntiles, gmax);
    const int CV = 2 * kMargin * k + 256;
    int NC = 1;
    while (NC < 2 * kMargin * k) NC <<= 1;
    NC = std::min(NC, 16 * 512);
    Sizer sz;
    sz.take<float>(static_cast<size_t>(s) * d);
    sz.take<float>(static_cast<size_t>(n) * kSeedRank);           // sample keys, by row
    sz.take<int64_t>(static_cast<size_t>(n) * kSeedRank);
    sz.take<float>(static_cast<size_t>(s_slots) * 128 * kSeedRank);  // sample search slots
    sz.take<int64_t>(static_cast<size_t>(s_slots) * 128 * kSeedRank);
    sz.take<float2>(static_cast<size_t>(l_slots) * 128 * CV);
    sz.take<int>(static_cast<size_t>(l_slots) * 128);
    sz.take<int>(static_cast<size_t>(n) + 1);                     // uncertified rows
    sz.take<float>(static_cast<size_t>(f_slots) * 128 * k);        // their list-path search
    sz.take<int64_t>(static_cast<size_t>(f_slots) * 128 * k);
    sz.take<float>(static_cast<size_t>(gmax) * 128 * k);
    sz.take<int32_t>(static_cast<size_t>(gmax) * 128 * k);
    // its own grow-only arena: the caller's search scratch (the tensor path's
    // lists and fallback list) is live while this runs
    ctx.s->xl.reserve(sz.used + 256);
    Carver cv{static_cast<char*>(ctx.s->xl.base())};
    float* Rs = cv.take<float>(static_cast<size_t>(s) * d);
    float* sk32 = cv.take<float>(static_cast<size_t>(n) * kSeedRank);
    int64_t* si32 = cv.take<int64_t>(static_cast<size_t>(n) * kSeedRank);
    float* spk = cv.take<float>(static_cast<size_t>(s_slots) * 128 * kSeedRank);
    int64_t* spi = cv.take<int64_t>(static_cast<size_t>(s_slots) * 128 * kSeedRank);
    float2* vlog = cv.take<float2>(static_cast<size_t>(l_slots) * 128 * CV);
    int* vlog_n = cv.take<int>(static_cast<size_t>(l_slots) * 128);
    int* fb = cv.take<int>(static_cast<size_t>(n) + 1);
    float* fpk = cv.take<float>(static_cast<size_t>(f_slots) * 128 * k);
    int64_t* fpi = cv.take<int64_t>(static_cast<size_t>(f_slots) * 128 * k);
    float* fgk = cv.take<float>(static_cast<size_t>(gmax) * 128 * k);
    int32_t* fgi = cv.take<int32_t>(static_cast<size_t>(gmax) * 128 * k);
    {
        ProfileScope ps(stream, "exact_large_sample");
        const int64_t tot = s * d;
        gather_strided_kernel<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, stream>>>(dR, d, stride, s, Rs);
        KNN_LAUNCH_CHECK();
    }
    ExactArgs sa{};  // the sample search (k' = 32, raw keys, rows of Q by the list)
    sa.Q = dQ;
    sa.R = Rs;
    sa.n = n;
    sa.m = s;
    sa.d = d;
    sa.k = kSeedRank;
    sa.ntiles = stiles;
    sa.qlist = qlist;
    sa.qcount = qcount;
    sa.raw_keys = 1;
    sa.out_key = sk32;
    sa.out_idx = si32;
    sa.part_key = spk;
    sa.part_idx = spi;
    launch_exact(metric, sa, stream);
    // 2. the threshold-log pass
    ExactArgs a{};
    a.Q = dQ;
    a.R = dR;
    a.n = n;
    a.m = m;
    a.d = d;
    a.k = k;
    a.ntiles = ntiles;
    a.qlist = qlist;
    a.qcount = qcount;
    a.t0 = sk32 + (kSeedRank - 1);
    a.t0_stride = kSeedRank;
    a.vlog = vlog;
    a.vlog_n = vlog_n;
    a.CV = CV;
    launch_exact_log(metric, a, stream);
    // 3. select
    KNN_CUDA_CHECK(cudaMemsetAsync(fb, 0, sizeof(int), stream));
    SelArgs sl{};
    sl.qlist = qlist;
    sl.qcount = qcount;
    sl.vlog = vlog;
    sl.vlog_n = vlog_n;
    sl.CV = CV;
    sl.NC = NC;
    sl.k = k;
    sl.n = n;
    sl.ntiles = ntiles;
    sl.max_ctas = lmax;
    sl.t0 = a.t0;
    sl.t0_stride = kSeedRank;
    sl.metric = metric;
    sl.raw_keys = raw_keys;
    sl.index_base = index_base;
    sl.out = d_out;
    sl.out_idx = d_idx;
    sl.fb_count = fb;
    sl.fb_list = fb + 1;
    {
        const int nt = NC <= 16 * 256 ? 256 : 512;
        const size_t smem = static_cast<size_t>(NC) * 8;
        auto kern = nt == 256 ? select_exact_kernel<256> : select_exact_kernel<512>;
        KNN_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            static_cast<int>(smem)));
        ProfileScope ps(stream, "select_exact_kernel");
        const int64_t grid = qcount ? std::min<int64_t>(n, 8 * kSmCount) : n;
        kern<<<static_cast<unsigned>(std::max<int64_t>(1, grid)), nt, smem, stream>>>(sl);
        KNN_LAUNCH_CHECK();
    }
    // 4. uncertified rows (a tail estimate of T0): the list path over the
    //    device-side row list (global lists), still on the device
    ExactArgs fa{};
    fa.Q = dQ;
    fa.R = dR;
    fa.n = n;
    fa.m = m;
    fa.d = d;
    fa.k = k;
    fa.ntiles = ntiles;
    fa.qlist = fb + 1;
    fa.qcount = fb;
    fa.index_base = index_base;
    fa.raw_keys = raw_keys;
    fa.out_key = d_out;
    fa.out_idx = d_idx;
    fa.part_key = fpk;
    fa.part_idx = fpi;
    fa.glist_key = fgk;
    fa.glist_idx = fgi;
    launch_exact(metric, fa, stream);
    if (fb_total) {  // chunked: accumulate the chunk's count
        add_count_kernel<<<1, 32, 0, stream>>>(fb_total, fb, first);
        KNN_LAUNCH_CHECK();
        return;
    }
    if (ctx.s->fb_dev)
        KNN_CUDA_CHECK(cudaMemcpyAsync(ctx.s->fb_dev, fb, sizeof(int), cudaMemcpyDeviceToDevice, stream));
    ctx.s->fb_on_device = true;
}

}  // namespace knnb200
