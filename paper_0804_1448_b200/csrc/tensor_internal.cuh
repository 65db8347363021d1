// tensor_internal.cuh -- shared pieces of the tensor path (L2, tcgen05):
// constants, per-query bound arithmetic, the kernel argument blocks, the
// filter CTA's pipeline roles and the launchers of the kernels that live in
// tensor_prep.cu, tensor_filter.cu, tensor_select.cu and tensor_rerank.cu.
// Orchestration: tensor_path.cu.  Design: DESIGN.md sec. 3.2-3.3 and 4.
#pragma once

#include <cuda.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdint>

#include "common.cuh"
#include "sm100.cuh"

namespace knnb200 {
namespace tp {

constexpr int TILE = 128;          // queries per MMA tile (M) and references per tile (N)
constexpr int EPI_WARPS = 8;       // two sets of four (one warp per TMEM lane quarter)
constexpr int EPI_THREADS = EPI_WARPS * 32;
constexpr int THREADS = 128 + EPI_THREADS;  // producer, MMA, TMEM-alloc, spare + epilogue
constexpr int KEXTRA = 0;          // bound list K' >= k + KEXTRA
constexpr int kLogGroups = 256;    // minimum logged candidate groups per (query, CTA part)
constexpr int kMaxLargeK = 1024;   // k > MAX_KQ: fixed-threshold filter + block selection
constexpr int MAX_KQ = 32;
constexpr int SMEM_LIMIT = 232448; // 227 KB opt-in per CTA

constexpr int RR_WARPS = 2;      // re-rank: warps (queries) per block
constexpr int RR_CAND = 128;     // exact candidates per query on the fast path (more: fallback)

struct Consts {         // per-query constants of the inclusion bound
    float nq;           // ||q~||^2
    float delta;        // delta_q + max_j delta_r
    float eps;          // accumulation error bound of A
    float c1;           // sqrt((1+rho)/(1-rho)), rounded up
};

// Rigorous inclusion threshold on A = ||r~||^2 - 2 q~.r~ given the k-th
// smallest A seen so far.  Any reference whose exact FP32
// key can still reach the final top-k has A <= thresh(A_k).  Rounded up.
__device__ __forceinline__ float thresh(float ak, const Consts& c) {
    const float u = sqrtf(fmaxf(ak + c.eps + c.nq, 0.f)) * (1.f + 1e-6f);
    const float v = c.c1 * (u + c.delta) + c.delta;
    const float t = v * v * (1.f + 4e-6f) - c.nq + c.eps;
    return t + fabsf(t) * 4e-6f + 1e-30f;
}

// Stream-K unit split of the filter: CTA c owns units [U c / G, U (c+1) / G)
// of the (query-tile pair, reference tile) sequence.
__device__ __forceinline__ int64_t unit_start(int64_t U, int G, int c) {
    return (U * c) / G;
}

__device__ __forceinline__ int first_cta_of(int64_t u0, int64_t U, int G) {
    int c = static_cast<int>((u0 * G) / U);
    while (c + 1 < G && unit_start(U, G, c + 1) <= u0) ++c;
    while (c > 0 && unit_start(U, G, c) > u0) --c;
    return c;
}

struct PrepArgs {
    const float* X;     // rows x d
    int64_t rows, rows_pad;
    int d, Kp;
    int norm_col;       // first of three folded-norm columns, -1 if not folded
    const float* mu;    // d
    const float* scale; // 1
    __half* Xh;         // rows_pad x Kp
    float* norm;        // refs, no-fold: ||r~||^2 per row (+inf padding)
    float4* qconst;     // queries: {nq, delta_q, ||q~||, 0}
    unsigned* gmax;     // refs: [0] max delta_r bits, [1] max ||r~|| bits
    unsigned* tinit;    // queries: per-row cross-CTA bound, set to "none" (0xffffffff)
    int* zero;          // queries: a counter cleared by block 0 (fallback count)
    int* pair_slots;    // queries: per query-tile pair, the number of CTAs touching it
    int pairs, G, rtiles;
    int64_t U;
};

// ordered-uint encoding of floats for atomicMin/Max over signed values
__device__ __forceinline__ unsigned enc(float f) {
    const unsigned u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float dec(unsigned u) {
    return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}
// 0xffffffff (memset "no bound yet") decodes as NaN: map it to +inf
__device__ __forceinline__ float dec_or_inf(unsigned u) {
    return fminf(kInf, dec(u));
}

struct FilterArgs {
    int64_t n, m;
    int qtiles, rtiles;
    int pairs;             // query-tile pairs (a CTA keeps both tiles of a pair resident)
    int64_t U;             // pairs * rtiles work units (one 128-reference tile x 256 queries)
    int G;                 // CTAs
    int S_max;             // partial-list slots per query tile
    int KB;                // 64-wide K blocks (full)
    int tail;              // 1: a narrow 16-wide K block follows (SWIZZLE_32B)
    int tile_bytes;        // bytes of one 128-row operand tile in shared memory
    int nslices;           // K / 16 MMA slices
    int stages;
    int k, Kq;
    int d;
    float gamma;           // accumulation error factor
    float c1;
    bool fold;
    const float4* qconst;
    const float* rnorm;    // no-fold norms
    const unsigned* gmax;
    unsigned* tglob;       // [n_pad] shared running threshold (ordered-uint, atomicMin)
    float* part_A;         // [parts][128][Kq] final bound list (keys) of each part
    int* part_cnt;         // [parts][128] entries in part_A
    int* log_n;            // [parts][128] groups logged (may exceed CG: overflow)
    float4* log_v;         // [parts][128][CG][2] the 8 A values of each logged group
    int2* log_h;           // [parts][128][CG] {group minimum bits, first reference index}
    int CG;                // log capacity (groups) per (part, query)
    int drain_at;          // drain when a lane holds this many group minima (<= CAP - 16)
    int mode;              // dev only (KNN_B200_FILTER_MODE): 0 full, 2 no epilogue work, 3 no pushes
    int dev_flags;         // dev only (KNN_B200_DEV_FLAGS): bit 0 MMA issuers spin instead of sleeping
    float* sink;
    unsigned long long* stats;  // dev only (KNN_B200_FILTER_STATS)
    // large-k (filter_fixed_kernel): seed tiles per segment, per-query
    // threshold T0, compact value log {A, reference index} of capacity CV
    int W;
    int seed_off;          // 0 / 1: interleaved seed tile positions (retry uses fresh tiles)
    int seed_rank;         // T0 = thresh(seed_rank-th smallest seed group minimum)
    int log_all;           // fixed filter: append without the per-chunk vote (dense logs)
    float* t0;             // [n_pad]
    float2* vlog;          // [parts][128][CV]
    int CV;
    const int* pair_slots;  // [pairs] CTAs touching each query-tile pair (query prep)
};

__device__ __forceinline__ Consts load_consts(const FilterArgs& a, int64_t q) {
    const float4 qc = a.qconst[q];
    const float dr = __uint_as_float(a.gmax[0]);
    const float rn = __uint_as_float(a.gmax[1]);
    Consts c;
    c.nq = qc.x;
    c.delta = (qc.y + dr) * (1.f + 1e-6f);
    // |A - (||r~||^2 - 2 q~.r~)| <= gamma * (2 ||q~|| ||r~|| + ||r~||^2)  (+ norm rounding
    // when the norm is added in fp32 instead of folded)
    const float mag = 2.f * qc.z * rn + rn * rn;
    c.eps = a.gamma * mag + (a.fold ? 0.f : 0x1.0p-22f * mag) + 1e-30f;
    c.c1 = a.c1;
    return c;
}

__device__ __forceinline__ float min3(float x, float y, float z) {
    float w;
    asm("min.f32 %0, %1, %2, %3;" : "=f"(w) : "f"(x), "f"(y), "f"(z));
    return w;
}

// Dev-only per-warp counters (make EXTRA=-DKNN_B200_FILTER_STATS, then run with
// KNN_B200_FILTER_STATS=1); compiled out of the product build.
#ifdef KNN_B200_FILTER_STATS
constexpr bool kStats = true;
#else
constexpr bool kStats = false;
#endif

#ifndef KNN_CAP
#define KNN_CAP 24
#endif
constexpr int CAP = KNN_CAP;   // per-lane buffered group minima awaiting the bound list (smem);
                               // drained once per tile (a tile pushes <= 16), off the TMEM path
constexpr int EPI_REGS = 232;  // setmaxnreg: epilogue warpgroups grow by what warpgroup 0 frees
// (the pool is the CTA's launch allocation: 2 x 128 x (232 - 168) = 128 x (168 - 40))
constexpr int CTRL_REGS = 40;

// Push of one 8-column group whose minimum is under the lane's bound: its 8
// values (32 B) and head {minimum, first column} at slot `off` of the query's
// log, the minimum into the lane's smem buffer (for the drain).  The stores
// are predicated in PTX (never a branch); the cursor updates stay in C++ so
// ptxas sees plain selects.  Capacity is checked once per unit by the caller.
template <int STRIDE>
__device__ __forceinline__ void push_group(float gm, float tf, uint32_t& sgp, int& off, float4* lvb,
                                           int2* lhb, const float* w, int col) {
    const bool hit = gm <= tf;
    // byte offsets from the per-lane bases: one wide multiply-add per address
    float4* pv = reinterpret_cast<float4*>(reinterpret_cast<char*>(lvb) + static_cast<uint64_t>(static_cast<uint32_t>(off)) * 32u);
    int2* ph = reinterpret_cast<int2*>(reinterpret_cast<char*>(lhb) + static_cast<uint64_t>(static_cast<uint32_t>(off)) * 8u);
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %0, 0;\n\t"
        "@p st.global.v8.f32 [%1], {%5, %6, %7, %8, %9, %10, %11, %12};\n\t"
        "@p st.global.v2.b32 [%2], {%3, %4};\n\t"
        "@p st.shared.f32 [%13], %3;\n\t}"
        :
        : "r"(static_cast<int>(hit)), "l"(pv), "l"(ph), "f"(gm), "r"(col), "f"(w[0]), "f"(w[1]),
          "f"(w[2]), "f"(w[3]), "f"(w[4]), "f"(w[5]), "f"(w[6]), "f"(w[7]), "r"(sgp)
        : "memory");
    off += hit ? 1 : 0;
    sgp += hit ? STRIDE : 0;
}

// no-fold layouts: add ||r~||^2 of 32 consecutive references to the raw -2 q~.r~,
// from the warp's shared-memory copy of the unit's norms (broadcast reads)
__device__ __forceinline__ void add_rnorm_smem(float (&v)[32], const float* rn) {
    const float4* nr = reinterpret_cast<const float4*>(rn);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const float4 w = nr[j];
        v[4 * j] += w.x;
        v[4 * j + 1] += w.y;
        v[4 * j + 2] += w.z;
        v[4 * j + 3] += w.w;
    }
}

__device__ __forceinline__ float lds_f32(uint32_t addr) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
    return v;
}

// 32-byte read-only global load (one full sector per lane: LDG.E.256)
__device__ __forceinline__ void ldg8(const float* p, float (&v)[8]) {
    asm volatile("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]),
                   "=f"(v[6]), "=f"(v[7])
                 : "l"(p));
}

// 256-bit load with an L2 eviction-priority policy (createpolicy operand)
__device__ __forceinline__ void ldg8_hint(const float* p, float (&v)[8], uint64_t pol) {
    asm volatile("ld.global.nc.L2::cache_hint.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8], %9;"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]),
                   "=f"(v[6]), "=f"(v[7])
                 : "l"(p), "l"(pol));
}

__device__ __forceinline__ int2 ldg2_hint(const int* p, uint64_t pol) {
    int2 v;
    asm volatile("ld.global.nc.L2::cache_hint.v2.b32 {%0, %1}, [%2], %3;" : "=r"(v.x), "=r"(v.y) : "l"(p), "l"(pol));
    return v;
}

__device__ __forceinline__ int ldg_hint(const int* p, uint64_t pol) {
    int v;
    asm volatile("ld.global.nc.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}

// read-once data (the group logs): evicted before the reference rows
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

// Exact FP32 key of one (query row, reference row) pair, key_step order.
// Rows 32-byte aligned (d % 8 == 0, 32-byte aligned bases): 256-bit loads.
__device__ __forceinline__ float exact_key_l2(const float* qrow, const float* rrow, int d) {
    float acc = 0.f;
    if ((d & 7) == 0 && ((reinterpret_cast<uintptr_t>(qrow) | reinterpret_cast<uintptr_t>(rrow)) & 31) == 0) {
#pragma unroll 4
        for (int c8 = 0; c8 < (d >> 3); ++c8) {
            float u[8], w[8];
            ldg8(qrow + 8 * c8, u);
            ldg8(rrow + 8 * c8, w);
#pragma unroll
            for (int e = 0; e < 8; ++e) acc = key_step<kL2>(acc, u[e], w[e]);
        }
    } else if ((d & 3) == 0) {
        const float4* q4 = reinterpret_cast<const float4*>(qrow);
        const float4* r4 = reinterpret_cast<const float4*>(rrow);
#pragma unroll 8
        for (int c4 = 0; c4 < (d >> 2); ++c4) {
            const float4 u = __ldg(q4 + c4), w = __ldg(r4 + c4);
            acc = key_step<kL2>(acc, u.x, w.x);
            acc = key_step<kL2>(acc, u.y, w.y);
            acc = key_step<kL2>(acc, u.z, w.z);
            acc = key_step<kL2>(acc, u.w, w.w);
        }
    } else {
        for (int cc = 0; cc < d; ++cc) acc = key_step<kL2>(acc, __ldg(qrow + cc), __ldg(rrow + cc));
    }
    return acc;
}

// The KR smallest group minima seen by this (query, CTA part), sorted
// ascending, keys only: the list exists to bound A_(k) (any k distinct
// references with A <= v prove A_(k) <= v); candidate identities live in the
// global group log, not here.
template <int KR>
struct RegList {
    float key[KR];
    int cnt;

    __device__ __forceinline__ void reset() {
#pragma unroll
        for (int s = 0; s < KR; ++s) key[s] = kInf;
        cnt = 0;
    }
    // Branch-free insert by rank: slot s becomes max(key[s-1], min(x, key[s]))
    // (= key[s-1] if x sorts before it, x if it lands here, else unchanged).
    // Every slot depends only on x and the old list: no serial chain.
    __device__ __forceinline__ void insert(float x) {
#pragma unroll
        for (int s = KR - 1; s > 0; --s) key[s] = fmaxf(key[s - 1], fminf(x, key[s]));
        key[0] = fminf(x, key[0]);
        cnt = min(cnt + 1, KR);
    }
    // insert that leaves cnt alone for +inf ("nothing to insert" in a SIMT round)
    __device__ __forceinline__ void insert_maybe(float x) {
#pragma unroll
        for (int s = KR - 1; s > 0; --s) key[s] = fmaxf(key[s - 1], fminf(x, key[s]));
        key[0] = fminf(x, key[0]);
        cnt = min(cnt + (x < kInf ? 1 : 0), KR);
    }
    // Batch insert of up to 8 values (+inf = none; nv finite), KR <= 24: sort
    // the batch (19-comparator network), then one bitonic merge of the list
    // (padded to 24) with the reversed batch, keeping the KR smallest --
    // ~170 min/max for 8 values where 8 rank inserts cost 8 x 2 KR.
    __device__ __forceinline__ void insert8(float (&b)[8], int nv) {
        static_assert(KR <= 24, "insert8: list + batch must fit a 32-wide network");
        auto ce = [](float& x, float& y) {
            const float lo = fminf(x, y), hi = fmaxf(x, y);
            x = lo;
            y = hi;
        };
        ce(b[0], b[1]); ce(b[2], b[3]); ce(b[4], b[5]); ce(b[6], b[7]);
        ce(b[0], b[2]); ce(b[1], b[3]); ce(b[4], b[6]); ce(b[5], b[7]);
        ce(b[1], b[2]); ce(b[5], b[6]); ce(b[0], b[4]); ce(b[3], b[7]);
        ce(b[1], b[5]); ce(b[2], b[6]);
        ce(b[1], b[4]); ce(b[3], b[6]);
        ce(b[2], b[4]); ce(b[3], b[5]);
        ce(b[3], b[4]);
        float c[32];
#pragma unroll
        for (int s = 0; s < 24; ++s) c[s] = s < KR ? key[s] : kInf;
#pragma unroll
        for (int u = 0; u < 8; ++u) c[24 + u] = b[7 - u];
#pragma unroll
        for (int i = 0; i < 16; ++i) ce(c[i], c[i + 16]);
#pragma unroll
        for (int st = 8; st > 0; st >>= 1) {
#pragma unroll
            for (int i = 0; i < 16; ++i)
                if ((i & st) == 0) ce(c[i], c[i + st]);
        }
        if (KR > 16) {  // the 8 smallest of the upper half, sorted
#pragma unroll
            for (int i = 0; i < 8; ++i) c[16 + i] = fminf(c[16 + i], c[24 + i]);
#pragma unroll
            for (int st = 4; st > 0; st >>= 1) {
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    if ((i & st) == 0) ce(c[16 + i], c[16 + i + st]);
            }
        }
#pragma unroll
        for (int s = 0; s < KR; ++s) key[s] = c[s];
        cnt = min(cnt + nv, KR);
    }
    // key[k-1] for a runtime k.  The select chain is opaque inline PTX: written
    // as plain C++ the compiler turns it back into key[k-1], a dynamic index
    // that demotes the whole list to local memory.
    __device__ __forceinline__ float kth(int k) const {
        float v = kInf;
#pragma unroll
        for (int s = 0; s < KR; ++s)
            asm("{\n\t.reg .pred p;\n\tsetp.eq.s32 p, %2, %3;\n\tselp.f32 %0, %1, %0, p;\n\t}"
                : "+f"(v)
                : "f"(key[s]), "r"(k - 1), "r"(s));
        return v;
    }
};

// The unit sequence every role of a filter CTA walks: its stream-K range
// [u_begin, u_end) of (query-tile pair, reference tile) units, split into
// segments of one pair each.  With W > 0 each segment is preceded by W "seed"
// units: reference tiles spread evenly over the pair's whole reference range
// (the large-k threshold estimate, filter_fixed_kernel).
struct UnitSeq {
    int64_t u, u_end, seg_end;
    int rtiles, W, seed_left, p, off;
    __device__ __forceinline__ void init(int64_t ub, int64_t ue, int rt, int w, int seed_off = 0) {
        u = ub;
        u_end = ue;
        rtiles = rt;
        W = w;
        off = seed_off;
        if (u < u_end) begin_seg();
    }
    __device__ __forceinline__ void begin_seg() {
        p = static_cast<int>(u / rtiles);
        seg_end = min(u_end, static_cast<int64_t>(p + 1) * rtiles);
        seed_left = W;
    }
    __device__ __forceinline__ bool more() const { return u < u_end; }
    __device__ __forceinline__ bool seed() const { return seed_left > 0; }
    __device__ __forceinline__ int tile() const {
        return seed_left > 0
                   ? static_cast<int>((2LL * (W - seed_left) + off) * rtiles / (2LL * W))
                   : static_cast<int>(u % rtiles);
    }
    __device__ __forceinline__ void next() {
        if (seed_left > 0) {
            --seed_left;
            return;
        }
        if (++u < u_end && u == seg_end) begin_seg();
    }
};

struct Pipe {  // one filter CTA's pipeline objects
    unsigned char* As;   // 2 query tiles
    unsigned char* Bs;   // stages x reference tile
    int KBB;             // bytes of one 128-row operand tile
    uint64_t *full, *empty, *a_full, *a_empty, *tfull, *tempty;
    uint32_t tmem;
};

// warp 0, one elected thread: TMA loads of the query-tile pair (once per
// segment) and of every unit's reference tile into the stage ring
__device__ __forceinline__ void producer_role(const CUtensorMap* tq, const CUtensorMap* tr,
                                              const CUtensorMap* tqt, const CUtensorMap* trt,
                                              const FilterArgs& a, const Pipe& P, int64_t ub,
                                              int64_t ue, int W) {
    sm100::tma_prefetch(tq);
    sm100::tma_prefetch(tr);
    if (a.tail) {
        sm100::tma_prefetch(tqt);
        sm100::tma_prefetch(trt);
    }
    int stage = 0;
    uint32_t phase = 0, a_par = 0;
    int cur_p = -1;
    UnitSeq sq;
    sq.init(ub, ue, a.rtiles, W, a.seed_off);
    for (; sq.more(); sq.next()) {
        if (sq.p != cur_p) {
            if (cur_p >= 0) {
                sm100::mbar_wait_sleep(P.a_empty, a_par);
                a_par ^= 1u;
            }
            sm100::mbar_expect_tx(P.a_full, static_cast<uint32_t>(2 * P.KBB));
            for (int g = 0; g < 2; ++g) {
                for (int kb = 0; kb < a.KB; ++kb)
                    sm100::tma_load_2d(P.As + g * P.KBB + kb * 16384, tq, P.a_full, kb * 64,
                                       (2 * sq.p + g) * TILE);
                if (a.tail)
                    sm100::tma_load_2d(P.As + g * P.KBB + a.KB * 16384, tqt, P.a_full, 0,
                                       (2 * sq.p + g) * TILE);
            }
            cur_p = sq.p;
        }
        sm100::mbar_wait_sleep(P.empty + stage, phase ^ 1u);
        sm100::mbar_expect_tx(P.full + stage, static_cast<uint32_t>(P.KBB));
        unsigned char* dst = P.Bs + stage * P.KBB;
        const int rt = sq.tile();
        for (int kb = 0; kb < a.KB; ++kb)
            sm100::tma_load_2d(dst + kb * 16384, tr, P.full + stage, kb * 64, rt * TILE);
        if (a.tail) sm100::tma_load_2d(dst + a.KB * 16384, trt, P.full + stage, 0, rt * TILE);
        if (++stage == a.stages) {
            stage = 0;
            phase ^= 1u;
        }
    }
}

// The MMA issuers wait with a suspend-time hint: a spinning issuer would take
// issue slots from the two epilogue warps sharing its SM sub-partition.
__device__ __forceinline__ void mma_wait(const FilterArgs& a, uint64_t* bar, uint32_t parity) {
    if (a.dev_flags & 1) sm100::mbar_wait(bar, parity);
    else sm100::mbar_wait_sleep(bar, parity);
}

// One elected thread per query tile g (warps 1 and 3): per unit an M=128
// N=128 MMA chain into TMEM buffer [g][unit parity].  Two issuers, so a slow
// epilogue group of one query tile never holds back the other tile's MMAs;
// each commits to the shared stage / A-tile barriers (arrival count 2).
__device__ __forceinline__ void mma_role(const FilterArgs& a, const Pipe& P, int64_t ub, int64_t ue,
                                         int W, int g) {
    const uint32_t idesc = sm100::idesc_f16_f32(TILE, TILE);
    int stage = 0;
    uint32_t phase = 0, a_par = 0;
    int cur_p = -1;
    int64_t t = 0;
    UnitSeq sq;
    sq.init(ub, ue, a.rtiles, W, a.seed_off);
    for (; sq.more(); sq.next(), ++t) {
        if (sq.p != cur_p) {
            if (cur_p >= 0) sm100::mma_commit(P.a_empty);
            mma_wait(a, P.a_full, a_par);
            a_par ^= 1u;
            cur_p = sq.p;
        }
        const int b = static_cast<int>(t & 1);
        const uint32_t tpar = static_cast<uint32_t>((t >> 1) & 1);
        mma_wait(a, P.full + stage, phase);
        sm100::tc_fence_after();
        const uint32_t b0 = sm100::smem_u32(P.Bs + stage * P.KBB);
        {
            mma_wait(a, P.tempty + 2 * g + b, tpar ^ 1u);
            sm100::tc_fence_after();
            const uint32_t a0 = sm100::smem_u32(P.As + g * P.KBB);
            const uint32_t dt = P.tmem + static_cast<uint32_t>((2 * g + b) * TILE);
            const int main_slices = a.tail ? a.nslices - 1 : a.nslices;
            for (int ks = 0; ks < main_slices; ++ks) {
                const uint32_t off = static_cast<uint32_t>((ks >> 2) * 16384 + (ks & 3) * 32);
                sm100::mma_f16_ss(dt, sm100::sdesc_k_sw128(a0 + off), sm100::sdesc_k_sw128(b0 + off),
                                  idesc, ks > 0 ? 1u : 0u);
            }
            if (a.tail) {  // the 16-wide folded-norm K block
                const uint32_t off = static_cast<uint32_t>(a.KB * 16384);
                sm100::mma_f16_ss(dt, sm100::sdesc_k_sw32(a0 + off), sm100::sdesc_k_sw32(b0 + off), idesc,
                                  main_slices > 0 ? 1u : 0u);
            }
            sm100::mma_commit(P.tfull + 2 * g + b);
        }
        sm100::mma_commit(P.empty + stage);
        if (++stage == a.stages) {
            stage = 0;
            phase ^= 1u;
        }
    }
}

struct LargeArgs {
    const float* Q;
    const float* R;
    int64_t n;
    int d, k, S_max, NC;     // NC: smem capacity (power of two)
    FilterArgs f;
    int raw_keys;
    int64_t index_base;
    float* out;
    int64_t* out_idx;
    int* fb_count;
    int* fb_list;
    int fb_offset;
};

struct RerankArgs {
    const float* Q;        // original fp32 n x d
    const float* R;        // original fp32 m x d
    int64_t n;
    int d, k, Kq, S_max;
    int rtiles;
    FilterArgs f;          // constants + partial lists
    int raw_keys;
    int64_t index_base;
    float* out;
    int64_t* out_idx;
    int* fb_count;
    int* fb_list;
    int fb_offset;         // added to the recorded query index (deferred fallbacks)
};


__host__ __device__ constexpr size_t rr_warp_bytes(int span, int k) {
    return ((static_cast<size_t>(span) * 4 + RR_CAND * 8 + static_cast<size_t>(k) * 4 + 15) / 16) * 16 +
           static_cast<size_t>(k) * 8 + RR_CAND * 4;
}

struct Layout {
    int d16, Kp, KB, norm_col, stages, Kq;
    bool fold;
    bool tail;        // fold with a narrow 16-wide K block (d16 a multiple of 64)
    int tile_bytes;   // shared-memory bytes of one 128-row operand tile
    size_t smem;
};

inline Layout layout_for(int d, int k) {
    Layout L{};
    L.d16 = (d + 15) / 16 * 16;
    // candidate list size = the register-list template size >= k.  Each query
    // has >= 2 partial lists and only ~k+3 candidates inside the final bound
    // (measured, tools/margin_stats.py), so a list of k overflows inside the
    // bound only in near-tie-heavy data -- which the certificate catches.
    const int want = std::min(k + KEXTRA, MAX_KQ);
    static const int sizes[] = {4, 8, 12, 16, 20, 24, 32};
    L.Kq = 32;
    for (int sz : sizes)
        if (sz >= want) {
            L.Kq = sz;
            break;
        }
    const int kb_plain = (L.d16 + 63) / 64;
    int kfold, ncol;
    if (L.d16 - d >= 3) {
        kfold = L.d16;
        ncol = d;
    } else {
        kfold = L.d16 + 16;
        ncol = L.d16;
    }
    const int kb_fold = (kfold + 63) / 64;
    // epilogue smem: group-minimum buffers + staged reference norms (no-fold)
    const size_t epi = static_cast<size_t>(EPI_THREADS) * CAP * 4 +
                       static_cast<size_t>(EPI_WARPS) * TILE * 4;
    const size_t fixed = epi + 1024 /*align*/ + 512 /*barriers*/;
    auto stages_for = [&](size_t per) {
        const long avail = static_cast<long>(SMEM_LIMIT) - static_cast<long>(fixed + 2 * per);
        return avail > 0 ? static_cast<int>(avail / static_cast<long>(per)) : 0;
    };
    // folded norms past a multiple of 64 columns: a narrow 16-wide K block
    // (SWIZZLE_32B) instead of a mostly empty 64-wide one
    const bool tail = kfold % 64 == 16;
    const size_t per_fold = tail ? static_cast<size_t>(kfold / 64) * 16384 + 4096
                                 : static_cast<size_t>(kb_fold) * 16384;
    if (kb_fold == kb_plain || stages_for(per_fold) >= 3) {
        L.fold = true;
        L.tail = tail;
        L.Kp = kfold;
        L.KB = tail ? kfold / 64 : kb_fold;
        L.norm_col = ncol;
        L.tile_bytes = static_cast<int>(per_fold);
    } else {
        L.fold = false;
        L.tail = false;
        L.Kp = L.d16;
        L.KB = kb_plain;
        L.norm_col = -1;
        L.tile_bytes = kb_plain * 16384;
    }
    L.stages = std::min(stages_for(static_cast<size_t>(L.tile_bytes)), 6);
    L.smem = fixed + static_cast<size_t>(L.tile_bytes) * (2 + L.stages);
    return L;
}

// launchers (ProfileScope names are the ones bench.py / tools report)
void launch_range(const float* X, int64_t rows, int d, unsigned* mn, unsigned* mx,
                  cudaStream_t stream);
void launch_scale(const unsigned* mn, const unsigned* mx, int d, int Kp, float* mu, float* scale,
                  unsigned* gmax, cudaStream_t stream);
void launch_convert(const PrepArgs& pr, bool query, cudaStream_t stream);
void launch_filter(int Kq, const CUtensorMap& tq, const CUtensorMap& tr, const CUtensorMap& tqt,
                   const CUtensorMap& trt, const FilterArgs& fa, int G, size_t smem, cudaStream_t stream);
void launch_filter_fixed(const CUtensorMap& tq, const CUtensorMap& tr, const CUtensorMap& tqt,
                         const CUtensorMap& trt, const FilterArgs& fa, int G, size_t smem,
                         cudaStream_t stream);
void launch_select_large(const LargeArgs& la, cudaStream_t stream);
void launch_rerank(const RerankArgs& ra, size_t smem, cudaStream_t stream);
}  // namespace tp
}  // namespace knnb200
