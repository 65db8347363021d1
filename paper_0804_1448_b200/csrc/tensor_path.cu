// tensor_path.cu -- orchestration of the tcgen05 path (L2, k <= 1024).
//
// Replaces the reference's distance fill + selection (paths relative to
// /root/reference/proj: src/bruteforce.cpp:23-38,81-96, include/knn/metric.hpp:22-29,
// src/topk.cpp:17-33) for the Euclidean metric with a GEMM-form filter on
// the 5th-generation tensor cores followed by an exact re-rank:
//
//  1. prep      (tensor_prep.cu) Q, R -> centred, power-of-two-scaled fp16
//               copies (K-major, K padded to 16) with the squared norm of
//               every rounded reference folded into three extra K columns, so
//               one tcgen05.mma chain yields  A = ||r~||^2 - 2 q~.r~ ; every
//               point's rounding radius for the certificate.  The reference
//               side is prepared once per reference set (TensorRefs).
//  2. filter    (tensor_filter.cu) persistent, warp-specialised, stream-K over
//               (query-tile pair, reference tile) units: a TMA producer, one
//               MMA issuer per query tile, 8 epilogue warps (thread = query
//               row) that take FMNMX3 group minima against the query's
//               running bound, keep a register list of the smallest group
//               minima and log every group under the bound (small k), or log
//               every value under a seeded fixed threshold (large k).
//  3. select    small k (tensor_rerank.cu): warp per query, bound from the
//               union of the part lists, certificate, exact FP32 keys of the
//               logged candidates, exact top-k.  Large k (tensor_select.cu):
//               block per query, radix select, exact keys, bitonic sort.
//  4. fallback  uncertified queries are recomputed by the exact SIMT kernel
//               on the device (query list and count in HBM, no host round
//               trip).  Results are bitwise identical to the exact path.
#include <cuda_fp16.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "engine.cuh"
#include "exact_kernel.cuh"
#include "profile.cuh"
#include "tensor_internal.cuh"
#include "tensor_path.cuh"
#include "tmap.cuh"

namespace knnb200 {

using namespace tp;

bool tensor_path_supported(int64_t n, int64_t m, int d, int k) {
    if (d < 1 || d > 128 || k < 1 || k > kMaxLargeK) return false;
    if (m < k || n < 1 || m > (1LL << 30)) return false;
    return layout_for(d, k).stages >= 2;
}

size_t tensor_refs_bytes(int64_t m, int d) {
    const Layout L = layout_for(d, 1);
    const int64_t m_pad = (m + TILE - 1) / TILE * TILE;
    Sizer sz;
    sz.take<__half>(static_cast<size_t>(m_pad) * L.Kp);
    sz.take<float>(static_cast<size_t>(m_pad));
    sz.take<unsigned>(2 * static_cast<size_t>(d) + 2);
    sz.take<float>(static_cast<size_t>(d) + 1);
    return sz.used + 256;
}

// Reference side of the tensor path, independent of the queries: per-dimension
// midrange centre and power-of-two scale of R, fp16 copy with the folded
// squared norms, rounding radii.  (The centre/scale only shape the fp16
// rounding: queries outside R's range round with their own, larger, delta and
// the certificate (sec. 4 of DESIGN.md) accounts for it; a query whose
// coordinates overflow fp16 yields no candidates and is recomputed exactly.)
void tensor_prep_refs(cudaStream_t stream, const float* dR, int64_t m, int d, void* mem,
                      TensorRefs& r) {
    const Layout L = layout_for(d, 1);
    r.dR = dR;
    r.m = m;
    r.d = d;
    r.m_pad = (m + TILE - 1) / TILE * TILE;
    Carver cv{static_cast<char*>(mem)};
    r.Rh = cv.take<__half>(static_cast<size_t>(r.m_pad) * L.Kp);
    r.rnorm = cv.take<float>(static_cast<size_t>(r.m_pad));
    unsigned* mnmx = cv.take<unsigned>(2 * static_cast<size_t>(d) + 2);
    r.mu = cv.take<float>(static_cast<size_t>(d) + 1);
    r.scale = r.mu + d;
    r.gmax = mnmx + 2 * d;
    KNN_CUDA_CHECK(cudaMemsetAsync(mnmx, 0xff, sizeof(unsigned) * d, stream));
    KNN_CUDA_CHECK(cudaMemsetAsync(mnmx + d, 0x00, sizeof(unsigned) * d, stream));
    launch_range(dR, m, d, mnmx, mnmx + d, stream);
    launch_scale(mnmx, mnmx + d, d, L.Kp, r.mu, r.scale, r.gmax, stream);
    PrepArgs pr{};
    pr.d = d;
    pr.Kp = L.Kp;
    pr.norm_col = L.fold ? L.norm_col : -1;
    pr.mu = r.mu;
    pr.scale = r.scale;
    pr.gmax = r.gmax;
    pr.X = dR;
    pr.rows = m;
    pr.rows_pad = r.m_pad;
    pr.Xh = r.Rh;
    pr.norm = r.rnorm;
    launch_convert(pr, false, stream);
}

void run_tensor_path(DeviceContext& ctx, cudaStream_t stream, const float* dQ, int64_t n,
                     const float* dR, int64_t m, int d, int k, int raw_keys, int64_t index_base,
                     float* d_out, int64_t* d_idx) {
    ctx.s->refs.reserve(tensor_refs_bytes(m, d));
    TensorRefs r;
    tensor_prep_refs(stream, dR, m, d, ctx.s->refs.base(), r);
    tensor_search(ctx, stream, r, dQ, n, k, raw_keys, index_base, d_out, d_idx);
}

void tensor_search(DeviceContext& ctx, cudaStream_t stream, const TensorRefs& refs,
                   const float* dQ, int64_t n, int k, int raw_keys, int64_t index_base,
                   float* d_out, int64_t* d_idx, const FallbackSink* sink, int margin) {
    const float* dR = refs.dR;
    const int64_t m = refs.m;
    const int d = refs.d;
    const Layout L = layout_for(d, k);
    const int pairs = static_cast<int>((n + 2 * TILE - 1) / (2 * TILE));
    const int qtiles = 2 * pairs;  // the last tile of the last pair may be all padding
    const int rtiles = static_cast<int>((m + TILE - 1) / TILE);
    const int64_t n_pad = static_cast<int64_t>(qtiles) * TILE;
    const int64_t m_pad = static_cast<int64_t>(rtiles) * TILE;
    const int64_t U = static_cast<int64_t>(pairs) * rtiles;
    const bool large = k > MAX_KQ;
    if (large)
        if (const char* e = std::getenv("KNN_B200_LARGE_MARGIN")) margin = std::max(1, std::atoi(e));  // dev
    // at most ~29 CTAs share a query-tile pair, so a query has <= 32 partial lists
    // CTAs per query-tile pair: at least ~6 units each (every CTA part of a
    // pair restarts its bound list, so short parts push most of their groups
    // and the re-rank merges more lists; config A, 4800^2: 6 per pair instead
    // of 8, filter + re-rank 70 -> 66 us); at most 29 (<= 32 list slots)
    int per_pair = std::max(1, std::min(29, rtiles / 6));
    if (const char* e = std::getenv("KNN_B200_CTAS_PER_PAIR")) per_pair = std::max(1, std::min(29, std::atoi(e)));  // dev
    const int G = static_cast<int>(std::min<int64_t>(std::min<int64_t>(kSmCount, U),
                                                     static_cast<int64_t>(pairs) * per_pair));
    // partial-list slots per query tile under the stream-K split
    int S_max = 1;
    for (int pp = 0; pp < pairs; ++pp) {
        const int64_t u0 = static_cast<int64_t>(pp) * rtiles, u1 = u0 + rtiles - 1;
        const int c0 = static_cast<int>((u0 * G) / U), c1 = static_cast<int>((u1 * G) / U);
        S_max = std::max(S_max, c1 - c0 + 3);  // +2 slack for floor rounding at the ends
    }
    if (S_max > 32) throw CudaError("tensor path: too many partial lists per query tile");
    const int64_t parts = static_cast<int64_t>(qtiles) * S_max;

    Sizer sz;
    sz.take<__half>(static_cast<size_t>(n_pad) * L.Kp);
    sz.take<float4>(static_cast<size_t>(n_pad));
    // group-log capacity: ~1.5x the expected number of running-bound records
    // of a whole pair stream, k (1 + ln(groups / k)), at least 256
    int CG = 0;
    if (!large) {
        const double recs = k * (1.0 + std::log(std::max(1.0, (m / 8.0) / k)));
        CG = kLogGroups;
        while (CG < 1.5 * recs && CG < 4096) CG *= 2;
    }
    // large k: T0 ~ the (2k)-th smallest A; log room for twice that per part
    const int CV = large ? 2 * margin * k + 256 : 0;
    const int64_t np_list = large ? 0 : parts;
    sz.take<float>(static_cast<size_t>(np_list) * L.Kq * TILE);
    sz.take<int>(static_cast<size_t>(parts) * TILE);
    sz.take<int>(static_cast<size_t>(parts) * TILE);
    sz.take<float4>(static_cast<size_t>(parts) * TILE * CG * 2);
    sz.take<int2>(static_cast<size_t>(parts) * TILE * CG);
    sz.take<int>(static_cast<size_t>(n) + 1);
    sz.take<unsigned>(static_cast<size_t>(n_pad));
    sz.take<float>(large ? static_cast<size_t>(n_pad) : 0);
    sz.take<float2>(static_cast<size_t>(parts) * TILE * CV);
    sz.take<int>(static_cast<size_t>(pairs));
    // small k: the certification fallback runs on the device (exact kernel over
    // the failed queries, count read on the device): its partial-list slots
    // the certification fallback runs on the device (exact kernel over the
    // failed queries, count read on the device): its partial-list slots, and
    // for k > 128 its global list scratch
    const size_t fb_part = fallback_part_elems(n, m, k);
    const size_t fb_glist = fallback_glist_elems(k);
    sz.take<float>(fb_part);
    sz.take<int64_t>(fb_part);
    sz.take<float>(fb_glist);
    sz.take<int32_t>(fb_glist);
    ctx.s->arena.reserve(sz.used + 256);
    Carver cv{static_cast<char*>(ctx.s->arena.base())};
    __half* Qh = cv.take<__half>(static_cast<size_t>(n_pad) * L.Kp);
    __half* Rh = refs.Rh;
    const float* rnorm = refs.rnorm;
    float4* qconst = cv.take<float4>(static_cast<size_t>(n_pad));
    float* part_A = cv.take<float>(static_cast<size_t>(np_list) * L.Kq * TILE);
    int* part_cnt = cv.take<int>(static_cast<size_t>(parts) * TILE);
    int* log_n = cv.take<int>(static_cast<size_t>(parts) * TILE);
    float4* log_v = cv.take<float4>(static_cast<size_t>(parts) * TILE * CG * 2);
    int2* log_h = cv.take<int2>(static_cast<size_t>(parts) * TILE * CG);
    int* fb = cv.take<int>(static_cast<size_t>(n) + 1);
    unsigned* tglob = cv.take<unsigned>(static_cast<size_t>(n_pad));
    float* t0 = cv.take<float>(large ? static_cast<size_t>(n_pad) : 0);
    float2* vlog = cv.take<float2>(static_cast<size_t>(parts) * TILE * CV);
    int* pair_slots = cv.take<int>(static_cast<size_t>(pairs));
    float* fb_pk = cv.take<float>(fb_part);
    int64_t* fb_pi = cv.take<int64_t>(fb_part);
    float* fb_gk = cv.take<float>(fb_glist);
    int32_t* fb_gi = cv.take<int32_t>(fb_glist);
    const unsigned* gmax = refs.gmax;

    // 1. per-search state and the query-side prep
    // (no memsets: the query conversion initialises the cross-CTA bounds and
    // the fallback counter; consumers read only the part slots a pair's CTAs
    // actually wrote)
    PrepArgs pr{};
    pr.d = d;
    pr.Kp = L.Kp;
    pr.norm_col = L.fold ? L.norm_col : -1;
    pr.mu = refs.mu;
    pr.scale = refs.scale;
    pr.gmax = nullptr;
    pr.X = dQ;
    pr.rows = n;
    pr.rows_pad = n_pad;
    pr.Xh = Qh;
    pr.qconst = qconst;
    pr.tinit = tglob;
    pr.zero = fb;
    pr.pair_slots = pair_slots;
    pr.pairs = pairs;
    pr.G = G;
    pr.rtiles = rtiles;
    pr.U = U;
    launch_convert(pr, true, stream);

    // 2. tcgen05 filter
    FilterArgs fa{};
    fa.n = n;
    fa.m = m;
    fa.qtiles = qtiles;
    fa.pairs = pairs;
    fa.rtiles = rtiles;
    fa.U = U;
    fa.G = G;
    fa.S_max = S_max;
    fa.KB = L.KB;
    fa.tail = L.tail ? 1 : 0;
    fa.tile_bytes = L.tile_bytes;
    fa.nslices = L.Kp / 16;
    fa.stages = L.stages;
    fa.k = k;
    fa.Kq = L.Kq;
    fa.d = d;
    // <= (slices + 4) roundings of 2^-23 relative to sum |terms| each, doubled
    fa.gamma = static_cast<float>((fa.nslices + 4) * std::ldexp(1.0, -21));
    const double rho = (d + 8) * std::ldexp(1.0, -24);
    fa.c1 = static_cast<float>(std::sqrt((1 + rho) / (1 - rho)) * (1 + 1e-6));
    fa.fold = L.fold;
    fa.qconst = qconst;
    fa.rnorm = rnorm;
    fa.gmax = gmax;
    fa.tglob = tglob;
    fa.part_A = part_A;
    fa.part_cnt = part_cnt;
    fa.log_n = log_n;
    fa.log_v = log_v;
    fa.log_h = log_h;
    fa.pair_slots = pair_slots;
    fa.CG = CG;
    if (const char* e = std::getenv("KNN_B200_FILTER_MODE")) fa.mode = std::atoi(e);
    if (const char* e = std::getenv("KNN_B200_DEV_FLAGS")) fa.dev_flags = std::atoi(e);
    fa.drain_at = 8;
    if (const char* e = std::getenv("KNN_B200_DRAIN_AT"))
        fa.drain_at = std::max(1, std::min(CAP - 16, std::atoi(e)));
    fa.sink = reinterpret_cast<float*>(log_n);
    const bool want_stats = kStats && std::getenv("KNN_B200_FILTER_STATS") != nullptr;
    if (want_stats) {
        KNN_CUDA_CHECK(cudaMallocAsync(&fa.stats, 8 * sizeof(unsigned long long), stream));
        KNN_CUDA_CHECK(cudaMemsetAsync(fa.stats, 0, 8 * sizeof(unsigned long long), stream));
    }
    const CUtensorMap tq = make_tmap_f16_sw128(Qh, n_pad, L.Kp, TILE, 64);
    const CUtensorMap tr = make_tmap_f16_sw128(Rh, m_pad, L.Kp, TILE, 64);
    // the narrow folded-norm K block (unused maps repeat the main ones)
    const CUtensorMap tqt = L.tail ? make_tmap_f16_tail16(Qh, n_pad, L.Kp, L.KB * 64, TILE) : tq;
    const CUtensorMap trt = L.tail ? make_tmap_f16_tail16(Rh, m_pad, L.Kp, L.KB * 64, TILE) : tr;
    if (large) {
        // seed: W tiles whose 32nd smallest group minimum estimates the
        // (margin*k)-th smallest A (rank ~ m * 32 / (128 W)), W >= 2
        fa.seed_rank = 32;
        // a warp's 32 queries x 32 columns hold ~1024 x (margin k) / m loggable
        // values: from ~6 on some query hits practically every chunk and the
        // vote only costs (config D: k = 100 / 256 filter 883 -> 859 / 793 ->
        // 775 us; at k = 33, ~2.6 expected, skipping it measured slower;
        // dev knob KNN_B200_LOG_ALL=0/1 overrides)
        fa.log_all = 1024.0 * margin * k / static_cast<double>(m) >= 6.0 ? 1 : 0;
        if (const char* e = std::getenv("KNN_B200_LOG_ALL")) fa.log_all = std::atoi(e) != 0;
        fa.W = static_cast<int>(std::min<int64_t>(
            rtiles, std::max<int64_t>(2, (m + 4LL * margin * k - 1) / (4LL * margin * k))));
        fa.seed_off = 0;
        fa.t0 = t0;
        fa.vlog = vlog;
        fa.CV = CV;
        // no epilogue buffers here: more stages, minus the staged reference norms
        int stages_fixed = std::min(L.stages + 2, 6);
        auto fixed_bytes = [&](int st) {
            return 1024 + 512 + static_cast<size_t>(EPI_WARPS) * TILE * 4 +
                   static_cast<size_t>(L.tile_bytes) * (2 + st);
        };
        while (stages_fixed > 2 && fixed_bytes(stages_fixed) > static_cast<size_t>(SMEM_LIMIT))
            --stages_fixed;
        const size_t smem_fixed = fixed_bytes(stages_fixed);
        fa.stages = stages_fixed;
        launch_filter_fixed(tq, tr, tqt, trt, fa, G, smem_fixed, stream);
        LargeArgs la{};
        la.Q = dQ;
        la.R = dR;
        la.n = n;
        la.d = d;
        la.k = k;
        la.S_max = S_max;
        // candidate capacity: values inside thresh(B) are ~1.1 k (B at most one
        // histogram bin above A_(k)); more -> the query takes the exact path
        int NC = 64;
        while (NC < k + k / 2 + 64) NC <<= 1;
        if (const char* e = std::getenv("KNN_B200_SELECT_NC_MULT"))  // dev
            NC *= std::max(1, std::atoi(e));
        la.NC = std::min(NC, 8192);
        la.f = fa;
        la.raw_keys = raw_keys;
        la.index_base = index_base;
        la.out = d_out;
        la.out_idx = d_idx;
        la.fb_count = sink ? sink->count : fb;
        la.fb_list = sink ? sink->list : fb + 1;
        la.fb_offset = sink ? sink->offset : 0;
        launch_select_large(la, stream);
    } else {
    launch_filter(L.Kq, tq, tr, tqt, trt, fa, G, L.smem, stream);
    }  // small k

    // 3. exact re-rank (small k; large k selected above)
    RerankArgs ra{};
    ra.Q = dQ;
    ra.R = dR;
    ra.n = n;
    ra.d = d;
    ra.k = k;
    ra.Kq = L.Kq;
    ra.S_max = S_max;
    ra.rtiles = rtiles;
    ra.f = fa;
    ra.raw_keys = raw_keys;
    ra.index_base = index_base;
    ra.out = d_out;
    ra.out_idx = d_idx;
    ra.fb_count = sink ? sink->count : fb;
    ra.fb_list = sink ? sink->list : fb + 1;
    ra.fb_offset = sink ? sink->offset : 0;
    const size_t rr_smem = static_cast<size_t>(RR_WARPS) * rr_warp_bytes(S_max * L.Kq, k);
    if (!large) launch_rerank(ra, rr_smem, stream);
    if (want_stats) {  // dev (make EXTRA=-DKNN_B200_FILTER_STATS): re-rank candidate counts
        unsigned long long h[8];
        KNN_CUDA_CHECK(cudaMemcpyAsync(h, fa.stats, sizeof(h), cudaMemcpyDeviceToHost, stream));
        KNN_CUDA_CHECK(cudaStreamSynchronize(stream));
        KNN_CUDA_CHECK(cudaFree(fa.stats));
        const double qn = std::max(1.0, static_cast<double>(h[2]));
        std::fprintf(stderr,
                     "[rerank stats] certified queries %.0f: candidates/query %.2f, in-tau groups/query "
                     "%.2f, logged groups/query %.2f, parts/query %.2f\n",
                     qn, h[0] / qn, h[1] / qn, h[3] / qn, h[4] / qn);
    }

    // 4. certification fallback (exact kernel on the failed queries), unless
    //    the caller collects them across several searches.
    if (sink) return;
    tensor_resolve_fallbacks(ctx, stream, refs, dQ, n, k, raw_keys, index_base, d_out, d_idx, fb,
                             fb_pk, fb_pi, fb_gk, fb_gi);
}

static bool fallback_smem_lists(int k) { return static_cast<size_t>(k) <= exact_smem_list_limit_k(); }

size_t fallback_part_elems(int64_t n, int64_t m, int k) {
    return static_cast<size_t>(exact_slots(n, exact_ntiles(m), exact_max_ctas(k, fallback_smem_lists(k)))) *
           exact_queries_per_cta() * k;
}

size_t fallback_glist_elems(int k) {
    return fallback_smem_lists(k) ? 0
                                  : static_cast<size_t>(exact_max_ctas(k, false)) * exact_queries_per_cta() * k;
}

void tensor_resolve_fallbacks(DeviceContext& ctx, cudaStream_t stream, const TensorRefs& refs,
                              const float* dQ, int64_t n, int k, int raw_keys, int64_t index_base,
                              float* d_out, int64_t* d_idx, int* fb, float* fb_pk, int64_t* fb_pi,
                              float* fb_gk, int32_t* fb_gi) {
    // On the device for every k: the exact kernel reads the failed query list
    // and its count from HBM (fixed grid), merge_exact finishes the blocks it
    // spread over several CTAs -- no host round trip, so the search stays
    // asynchronous and graph-capturable.  Large k on a large reference set:
    // the exact path's threshold-log selection over the same list.
    if (exact_large_applies(refs.m, k)) {
        run_exact_large(ctx, stream, dQ, n, refs.dR, refs.m, refs.d, k, kL2, raw_keys, index_base, d_out,
                        d_idx, fb + 1, fb);
        // the count the caller reads is the tensor path's (fb), not the
        // nested selection's
        if (ctx.s->fb_dev)
            KNN_CUDA_CHECK(cudaMemcpyAsync(ctx.s->fb_dev, fb, sizeof(int), cudaMemcpyDeviceToDevice, stream));
        ctx.s->fb_on_device = true;
        return;
    }
    ExactArgs ea{};
    ea.Q = dQ;
    ea.R = refs.dR;
    ea.n = n;
    ea.m = refs.m;
    ea.d = refs.d;
    ea.k = k;
    ea.ntiles = exact_ntiles(refs.m);
    ea.qlist = fb + 1;
    ea.qcount = fb;
    ea.index_base = index_base;
    ea.raw_keys = raw_keys;
    ea.out_key = d_out;
    ea.out_idx = d_idx;
    ea.part_key = fb_pk;
    ea.part_idx = fb_pi;
    if (fallback_glist_elems(k) > 0) {  // k > 128: lists in global memory
        ea.glist_key = fb_gk;
        ea.glist_idx = fb_gi;
    }
    launch_exact(kL2, ea, stream);
    if (ctx.s->fb_dev)
        KNN_CUDA_CHECK(cudaMemcpyAsync(ctx.s->fb_dev, fb, sizeof(int), cudaMemcpyDeviceToDevice, stream));
    ctx.s->fb_on_device = true;
}

}  // namespace knnb200
