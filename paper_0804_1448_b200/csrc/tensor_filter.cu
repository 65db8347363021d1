// tensor_filter.cu -- the persistent tcgen05 filter kernels: the running-bound
// filter of the small-k path (bound lists + group log) and the fixed-threshold
// filter of the large-k path (seed tiles + value log).  DESIGN.md sec. 3.2-3.3.
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdio>

#include "common.cuh"
#include "profile.cuh"
#include "sm100.cuh"
#include "tensor_internal.cuh"

namespace knnb200 {
namespace tp {

namespace {

#ifndef KNN_BATCH_MIN
#define KNN_BATCH_MIN 5  // rounds left for a batch (fewer: one rank insert per round)
#endif
#ifndef KNN_DRAIN_BATCH
#define KNN_DRAIN_BATCH 1  // 0: drains insert one buffered minimum per round (dev A/B)
#endif

// Dev-only filter modes (KNN_B200_FILTER_MODE: 2 no epilogue work, 3 no pushes,
// used to measure floors); compiled out of the product build, where the hot
// loop carries no mode checks.
#ifdef KNN_B200_DEV_MODES
__device__ __forceinline__ int kMode(const FilterArgs& a) { return a.mode; }
#else
__device__ __forceinline__ constexpr int kMode(const FilterArgs&) { return 0; }
#endif

// Persistent tcgen05 filter.  A work unit is one 128-reference tile against a
// resident PAIR of 128-query tiles: warp 0 streams reference tiles by TMA;
// one thread of warp 1 (query tile 0) and one of warp 3 (query tile 1) issue
// the M=128 N=128 MMA chain of their tile into TMEM buffer (g, unit parity);
// warp 2 owns the TMEM allocation.  Epilogue set g -- 4 warps, one per TMEM
// lane quarter -- reads both parity buffers of its tile in turn: thread =
// query row, 128 columns per unit in four 32-column chunks (one TMEM load in
// flight ahead of the scan).  Each query keeps one bound list per CTA part;
// pushed groups go to the global group log, their minima to a shared-memory
// buffer that the drain inserts into the list once per tile.
template <int KR, bool FOLD>
__global__ void __launch_bounds__(THREADS, 1)
    filter_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tr,
                  const __grid_constant__ CUtensorMap tqt, const __grid_constant__ CUtensorMap trt,
                  FilterArgs a) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1024-B aligned start, derived by offset so the compiler keeps the shared
    // address space (LDS/STS instead of generic accesses)
    unsigned char* base = smem_raw + ((1024u - (sm100::smem_u32(smem_raw) & 1023u)) & 1023u);
    const int KBB = a.tile_bytes;  // bytes of one 128-row operand tile
    unsigned char* As = base;                // 2 query tiles
    unsigned char* Bs = base + 2 * KBB;      // stages x reference tile
    float* GB = reinterpret_cast<float*>(Bs + a.stages * KBB);        // [CAP][512] group minima
    float* RN = GB + CAP * EPI_THREADS;  // [EPI_WARPS][128] staged ||r~||^2 (no-fold)
    uint64_t* bars = reinterpret_cast<uint64_t*>(RN + EPI_WARPS * TILE);
    uint64_t* full = bars;
    uint64_t* empty = bars + a.stages;
    uint64_t* a_full = bars + 2 * a.stages;
    uint64_t* a_empty = a_full + 1;
    uint64_t* tfull = a_full + 2;  // [query tile][parity]
    uint64_t* tempty = tfull + 4;  // [query tile][parity]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 4);

    // warp index via a shuffle: ptxas then knows it is warp-uniform and keeps
    // role-branch state (e.g. the global memory descriptor) in uniform registers
    const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
    const int lane = threadIdx.x & 31;
    const int cta = blockIdx.x;
    const int64_t u_begin = unit_start(a.U, a.G, cta);
    const int64_t u_end = unit_start(a.U, a.G, cta + 1);

    if (threadIdx.x == 0) {
        for (int s = 0; s < a.stages; ++s) {
            sm100::mbar_init(full + s, 1);
            sm100::mbar_init(empty + s, 2);
        }
        sm100::mbar_init(a_full, 1);
        sm100::mbar_init(a_empty, 2);
        for (int b = 0; b < 4; ++b) {
            sm100::mbar_init(tfull + b, 1);
            sm100::mbar_init(tempty + b, 4);
        }
        sm100::fence_mbar_init();
    }
    if (warp == 2) sm100::tmem_alloc(tmem_slot, 512);
    sm100::tc_fence_before();
    __syncthreads();
    sm100::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    sm100::pdl_wait();  // the query prep (the predecessor) is complete from here on

    if (warp < 4) sm100::reg_dealloc<CTRL_REGS>();
    const Pipe P{As, Bs, KBB, full, empty, a_full, a_empty, tfull, tempty, tmem};
    if (warp == 0) {
        if (sm100::elect_one()) producer_role(&tq, &tr, &tqt, &trt, a, P, u_begin, u_end, 0);
    } else if (warp == 1) {
        if (sm100::elect_one()) mma_role(a, P, u_begin, u_end, 0, 0);
    } else if (warp == 3) {
        if (sm100::elect_one()) mma_role(a, P, u_begin, u_end, 0, 1);
    } else if (warp >= 4) {
        // ------------------------------------------------- epilogue -------
        sm100::reg_alloc<EPI_REGS>();
        const int ew = warp - 4;          // 0..7
        const int grp = ew >> 2;          // query tile of the pair
        const int quarter = warp & 3;     // TMEM lane quarter
        const int et = ew * 32 + lane;    // buffer column (0..255)
        const int row = quarter * 32 + lane;
        const int k = a.k;
        const uint32_t sg0 = sm100::smem_u32(GB) + static_cast<uint32_t>(et) * 4;

        RegList<KR> L;
        L.reset();
        int cur_p = -1;
        uint32_t sgp = sg0;  // next buffer slot: (sgp - sg0) / (4 EPI_THREADS) minima buffered
        float T = kInf;      // own bound: thresh(k-th smallest group minimum of this list)
        float Tf = kInf;     // filter bound: min over every valid bound for this query
        float tfp = kInf;    // push bound: Tf, or -inf once the log is (nearly) full
        unsigned tg_pref = 0xffffffffu;  // prefetched cross-CTA bound (ordered uint)
        Consts qc{};
        int q = 0;
        int part = 0;
        float4* lvb = nullptr;  // this (query, part)'s group log: values, heads
        int2* lhb = nullptr;
        int ln = 0;             // groups logged so far

        // Drain: one buffered group minimum per lane per round into the bound
        // list, then refresh the bound from this list and other CTAs' lists
        // (global atomicMin, read one drain late so the load latency hides).
#define KNN_DRAIN()                                                                              \
    do {                                                                                         \
        const int nb = static_cast<int>((sgp - sg0) / (EPI_THREADS * 4));                       \
        const int mx_ = __reduce_max_sync(0xffffffffu, nb);                                      \
        int j_ = 0;                                                                              \
        /* five or more rounds left: batches of 8 through the merge network */                 \
        if constexpr (KNN_DRAIN_BATCH && KR <= 24) {                                             \
            _Pragma("unroll 1") for (; j_ + KNN_BATCH_MIN - 1 < mx_; j_ += 8) {                  \
                float b_[8];                                                                     \
                int nv_ = 0;                                                                     \
                _Pragma("unroll") for (int u_ = 0; u_ < 8; ++u_) {                               \
                    float g_ = j_ + u_ < nb ? lds_f32(sg0 + (j_ + u_) * (EPI_THREADS * 4)) : kInf; \
                    g_ = g_ <= Tf && g_ < L.key[KR - 1] ? g_ : kInf;                             \
                    b_[u_] = g_;                                                                 \
                    nv_ += g_ < kInf ? 1 : 0;                                                    \
                }                                                                                \
                if (__any_sync(0xffffffffu, nv_ > 0)) L.insert8(b_, nv_);                        \
            }                                                                                    \
        }                                                                                        \
        _Pragma("unroll 1") for (; j_ < mx_; ++j_) {                                             \
            const float g_ = j_ < nb ? lds_f32(sg0 + j_ * (EPI_THREADS * 4)) : kInf;             \
            /* a minimum at or above the list's last entry changes nothing */                  \
            if (__any_sync(0xffffffffu, g_ <= Tf && g_ < L.key[KR - 1])) L.insert(g_);           \
        }                                                                                        \
        sgp = sg0;                                                                               \
        if (L.cnt >= k) {                                                                        \
            const float tn_ = thresh(k == KR ? L.key[KR - 1] : L.kth(k), qc);                    \
            if (tn_ < T) {                                                                       \
                T = tn_;                                                                         \
                atomicMin(a.tglob + q, enc(T));                                                  \
            }                                                                                    \
        }                                                                                        \
        Tf = fminf(T, dec_or_inf(tg_pref));                                                      \
        tg_pref = __ldcg(a.tglob + q);                                                           \
    } while (0)

#define KNN_FLUSH()                                                                              \
    do {                                                                                         \
        /* row-major per query ([part][row][Kq]): the re-rank reads a list */                 \
        /* with one coalesced load instead of Kq lines */                                       \
        float* pa_ = a.part_A + (static_cast<int64_t>(part) * TILE + row) * a.Kq;                \
        _Pragma("unroll") for (int e_ = 0; e_ < KR; ++e_)                                        \
            if (e_ < L.cnt) pa_[e_] = L.key[e_];                                                 \
        a.part_cnt[part * TILE + row] = L.cnt;                                                   \
        a.log_n[part * TILE + row] = ln > a.CG - 16 ? a.CG + 1 : ln; /* (nearly) full: overflow */ \
    } while (0)

        // One 32-column chunk, branch-free: the FMNMX3 minimum of each 8-column
        // group; if some lane of the warp has a group under its bound, all four
        // groups are pushed with predicated stores (a hit must not cost a
        // divergent branch: with 32 queries per warp most chunks hit).
#define KNN_SCAN32(rr, colb)                                                                     \
    do {                                                                                         \
        float v_[32];                                                                            \
        _Pragma("unroll") for (int j_ = 0; j_ < 32; ++j_) v_[j_] = __uint_as_float(rr[j_]);      \
        if (!FOLD) add_rnorm_smem(v_, rnw + ((colb) - col_base));                              \
        float gm_[4];                                                                            \
        _Pragma("unroll") for (int i_ = 0; i_ < 4; ++i_) {                                       \
            const float* w_ = v_ + 8 * i_;                                                       \
            gm_[i_] = fminf(min3(min3(w_[0], w_[1], w_[2]), min3(w_[3], w_[4], w_[5]), w_[6]),   \
                            w_[7]);                                                              \
        }                                                                                        \
        if (kMode(a) != 3 &&                                                                       \
            __any_sync(0xffffffffu, fminf(fminf(gm_[0], gm_[1]), fminf(gm_[2], gm_[3])) <= tfp)) { \
            _Pragma("unroll") for (int i_ = 0; i_ < 4; ++i_)                                     \
                push_group<EPI_THREADS * 4>(gm_[i_], tfp, sgp, ln, lvb, lhb, v_ + 8 * i_,        \
                                            (colb) + 8 * i_);                                    \
        }                                                                                        \
    } while (0)

        int p = static_cast<int>(u_begin / a.rtiles);
        int rt = static_cast<int>(u_begin % a.rtiles);
        const int nunits = static_cast<int>(u_end - u_begin);
        const uint32_t tlane = tmem + (static_cast<uint32_t>(quarter * 32) << 16) +
                               static_cast<uint32_t>(2 * grp * TILE);
        auto wait_full = [&](int t) {
            sm100::mbar_wait(tfull + 2 * grp + (t & 1), static_cast<uint32_t>((t >> 1) & 1));
            sm100::tc_fence_after();
        };
        auto release = [&](int t) {
            sm100::tc_fence_before();
            __syncwarp();
            if (lane == 0) sm100::mbar_arrive(tempty + 2 * grp + (t & 1));
        };

        // Software pipeline over 32-column chunks, one TMEM load in flight
        // (tcgen05.wait::ld waits for all): the load of chunk c+1 -- chunk 0
        // of the next tile after chunk 3 -- overlaps the scan of chunk c.
        uint32_t ra[32], rb[32];
        if (kMode(a) != 2 && nunits > 0) {
            wait_full(0);
            sm100::tmem_ld_32x32b_x32(tlane, ra);
            sm100::tmem_ld_wait();
        }
        // no-fold layouts: the unit's 128 reference norms are staged in this
        // warp's smem slot (one 16-B load per lane, issued a unit ahead) and
        // read back as broadcasts, instead of 8 global loads per chunk
        float* const rnw = RN + ew * TILE;
        float4 rn_nx = make_float4(0.f, 0.f, 0.f, 0.f);
        if (!FOLD && nunits > 0)
            rn_nx = __ldg(reinterpret_cast<const float4*>(a.rnorm + rt * TILE) + lane);
        for (int t = 0; t < nunits; ++t) {
            if (p != cur_p) {
                if (cur_p >= 0) {
                    KNN_DRAIN();
                    KNN_FLUSH();
                }
                cur_p = p;
                const int qt = 2 * p + grp;
                q = qt * TILE + row;
                const int slot = cta - first_cta_of(static_cast<int64_t>(p) * a.rtiles, a.U, a.G);
                part = qt * a.S_max + slot;
                const int64_t lq = (static_cast<int64_t>(part) * TILE + row) * a.CG;
                lvb = a.log_v + 2 * lq;
                lhb = a.log_h + lq;
                ln = 0;
                qc = load_consts(a, q);
                L.reset();
                T = kInf;
                tg_pref = __ldcg(a.tglob + q);
                Tf = dec_or_inf(tg_pref);
                sgp = sg0;
            }
            // a unit pushes <= 16 groups: stop pushing (the query then fails the
            // certificate and is recomputed exactly) once fewer slots are left
            tfp = ln > a.CG - 16 ? -kInf : Tf;
            const int col_base = rt * TILE;
            const uint32_t taddr = tlane + static_cast<uint32_t>((t & 1) * TILE);
            if (!FOLD) {  // stage this unit's norms, prefetch the next unit's
                __syncwarp();
                reinterpret_cast<float4*>(rnw)[lane] = rn_nx;
                __syncwarp();
                if (t + 1 < nunits) {
                    const int nrt = rt + 1 == a.rtiles ? 0 : rt + 1;
                    rn_nx = __ldg(reinterpret_cast<const float4*>(a.rnorm + nrt * TILE) + lane);
                }
            }
            if (kMode(a) == 2) {
                wait_full(t);
                release(t);
            } else {
                sm100::tmem_ld_32x32b_x32(taddr + 32, rb);
                KNN_SCAN32(ra, col_base);
                sm100::tmem_ld_wait();
                sm100::tmem_ld_32x32b_x32(taddr + 64, ra);
                KNN_SCAN32(rb, col_base + 32);
                sm100::tmem_ld_wait();
                sm100::tmem_ld_32x32b_x32(taddr + 96, rb);
                KNN_SCAN32(ra, col_base + 64);
                sm100::tmem_ld_wait();
                release(t);  // all four chunks of tile t are in registers
                KNN_SCAN32(rb, col_base + 96);
                // drain after the release, so the MMA never waits on the list
                if (__any_sync(0xffffffffu, sgp - sg0 >= static_cast<uint32_t>(a.drain_at * EPI_THREADS * 4)))
                    KNN_DRAIN();
                if (t + 1 < nunits) {
                    wait_full(t + 1);
                    sm100::tmem_ld_32x32b_x32(tlane + static_cast<uint32_t>(((t + 1) & 1) * TILE), ra);
                    sm100::tmem_ld_wait();
                }
            }
            if (++rt == a.rtiles) {
                rt = 0;
                ++p;
            }
        }
        if (cur_p >= 0) {
            KNN_DRAIN();
            KNN_FLUSH();
        }
#undef KNN_SCAN32
#undef KNN_DRAIN
#undef KNN_FLUSH
    }

    sm100::pdl_trigger();
    sm100::tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        sm100::tc_fence_after();
        sm100::tmem_dealloc(tmem, 512);
    }
}

// Large k (k > 32): one filter pass with a FIXED per-query threshold.  Each
// segment starts with W seed units (reference tiles spread over the pair's
// whole reference range, filter_fixed_kernel only): every group minimum of
// the seed goes into a 32-entry list and T0 = thresh(list[seed_rank-1]) is an
// estimate of thresh(A_(c*k)).  The main units then log every value A <= T0
// (compact {A, index} records, predicated stores).  T0 is only an estimate;
// the selection kernel certifies it (at least k logged values and
// thresh(A_(k)) <= T0, no log overflow) and sends the rest to the exact path.
template <bool FOLD>
__global__ void __launch_bounds__(THREADS, 1)
    filter_fixed_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tr,
                        const __grid_constant__ CUtensorMap tqt, const __grid_constant__ CUtensorMap trt,
                        FilterArgs a) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* base = smem_raw + ((1024u - (sm100::smem_u32(smem_raw) & 1023u)) & 1023u);
    const int KBB = a.tile_bytes;
    unsigned char* As = base;
    unsigned char* Bs = base + 2 * KBB;
    float* RN = reinterpret_cast<float*>(Bs + a.stages * KBB);  // [EPI_WARPS][128] staged norms
    uint64_t* bars = reinterpret_cast<uint64_t*>(RN + EPI_WARPS * TILE);
    uint64_t* full = bars;
    uint64_t* empty = bars + a.stages;
    uint64_t* a_full = bars + 2 * a.stages;
    uint64_t* a_empty = a_full + 1;
    uint64_t* tfull = a_full + 2;
    uint64_t* tempty = tfull + 4;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 4);

    // warp index via a shuffle: ptxas then knows it is warp-uniform and keeps
    // role-branch state (e.g. the global memory descriptor) in uniform registers
    const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
    const int lane = threadIdx.x & 31;
    const int cta = blockIdx.x;
    const int64_t u_begin = unit_start(a.U, a.G, cta);
    const int64_t u_end = unit_start(a.U, a.G, cta + 1);

    if (threadIdx.x == 0) {
        for (int s = 0; s < a.stages; ++s) {
            sm100::mbar_init(full + s, 1);
            sm100::mbar_init(empty + s, 2);
        }
        sm100::mbar_init(a_full, 1);
        sm100::mbar_init(a_empty, 2);
        for (int b = 0; b < 4; ++b) {
            sm100::mbar_init(tfull + b, 1);
            sm100::mbar_init(tempty + b, 4);
        }
        sm100::fence_mbar_init();
    }
    if (warp == 2) sm100::tmem_alloc(tmem_slot, 512);
    sm100::tc_fence_before();
    __syncthreads();
    sm100::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    sm100::pdl_wait();  // the query prep (the predecessor) is complete from here on

    if (warp < 4) sm100::reg_dealloc<CTRL_REGS>();
    const Pipe P{As, Bs, KBB, full, empty, a_full, a_empty, tfull, tempty, tmem};
    if (warp == 0) {
        if (sm100::elect_one()) producer_role(&tq, &tr, &tqt, &trt, a, P, u_begin, u_end, a.W);
    } else if (warp == 1) {
        if (sm100::elect_one()) mma_role(a, P, u_begin, u_end, a.W, 0);
    } else if (warp == 3) {
        if (sm100::elect_one()) mma_role(a, P, u_begin, u_end, a.W, 1);
    } else if (warp >= 4) {
        sm100::reg_alloc<EPI_REGS>();
        const int ew = warp - 4;
        const int grp = ew >> 2;
        const int quarter = warp & 3;
        const int row = quarter * 32 + lane;
        const uint32_t tlane = tmem + (static_cast<uint32_t>(quarter * 32) << 16) +
                               static_cast<uint32_t>(2 * grp * TILE);
        RegList<32> S;  // seed: the 32 smallest seed group minima
        S.reset();
        float T0 = kInf;   // the segment's fixed threshold (after its seed units)
        float tlog = kInf; // T0, or -inf once the log is (nearly) full
        Consts qc{};
        int64_t q = 0, part = 0;
        float2* vlp = nullptr;
        int ln = 0;
        int cur_p = -1;
        bool was_seed = false;
        int64_t t = 0;
        UnitSeq sq;
        sq.init(u_begin, u_end, a.rtiles, a.W, a.seed_off);
        float* const rnw = RN + (warp - 4) * TILE;
        float4 rn_nx = make_float4(0.f, 0.f, 0.f, 0.f);
        if (!FOLD && sq.more())
            rn_nx = __ldg(reinterpret_cast<const float4*>(a.rnorm + sq.tile() * TILE) + lane);
        auto finish = [&]() { a.log_n[part * TILE + row] = ln; };

        // Log every value of a 32-column chunk at or under tlog: if some lane of
        // the warp has a value there, 3-instruction predicated appends of all 32
        // ({A, index} records, the cursor advanced in the same PTX block).
#define KNN_LOG32(rr, colb)                                                                      \
    do {                                                                                         \
        float v_[32];                                                                            \
        _Pragma("unroll") for (int j_ = 0; j_ < 32; ++j_) v_[j_] = __uint_as_float(rr[j_]);      \
        if (!FOLD) add_rnorm_smem(v_, rnw + ((colb) - col_base));                                \
        /* log_all: nearly every chunk has a loggable value for some query of */               \
        /* the warp (dense logs), so the minimum tree and vote are skipped */                   \
        bool go_ = a.log_all != 0;                                                               \
        if (!go_) {                                                                              \
            float m_[11];                                                                        \
            _Pragma("unroll") for (int i_ = 0; i_ < 10; ++i_)                                    \
                m_[i_] = min3(v_[3 * i_], v_[3 * i_ + 1], v_[3 * i_ + 2]);                       \
            m_[10] = fminf(v_[30], v_[31]);                                                      \
            const float cm_ = min3(min3(m_[0], m_[1], m_[2]), min3(m_[3], m_[4], m_[5]),         \
                                   min3(min3(m_[6], m_[7], m_[8]), m_[9], m_[10]));              \
            go_ = __any_sync(0xffffffffu, cm_ <= tlog);                                          \
        }                                                                                        \
        if (go_) {                                                                               \
            float2* const v0_ = vlp;                                                             \
            _Pragma("unroll") for (int e_ = 0; e_ < 32; ++e_)                                    \
                asm volatile(                                                                    \
                    "{\n\t.reg .pred p;\n\t"                                                     \
                    "setp.le.f32 p, %1, %2;\n\t"                                                 \
                    "@p st.global.v2.b32 [%0], {%1, %3};\n\t"                                    \
                    "@p add.s64 %0, %0, 8;\n\t}"                                                 \
                    : "+l"(vlp)                                                                  \
                    : "f"(v_[e_]), "f"(tlog), "r"((colb) + e_)                                   \
                    : "memory");                                                                 \
            ln += static_cast<int>(vlp - v0_);                                                   \
        }                                                                                        \
    } while (0)

        uint32_t ra[32], rb[32];
        for (; sq.more(); sq.next(), ++t) {
            if (sq.p != cur_p) {
                if (cur_p >= 0) finish();
                cur_p = sq.p;
                const int qt = 2 * sq.p + grp;
                q = static_cast<int64_t>(qt) * TILE + row;
                const int slot = cta - first_cta_of(static_cast<int64_t>(sq.p) * a.rtiles, a.U, a.G);
                part = static_cast<int64_t>(qt) * a.S_max + slot;
                vlp = a.vlog + (part * TILE + row) * a.CV;
                ln = 0;
                qc = load_consts(a, q);
                S.reset();
                T0 = kInf;
            }
            const bool seed = sq.seed();
            if (!seed && was_seed) {  // seed complete: fix the segment's threshold
                T0 = thresh(S.kth(a.seed_rank), qc);
                a.t0[q] = T0;  // identical from every CTA of the pair
            }
            was_seed = seed;
            const int b = static_cast<int>(t & 1);
            sm100::mbar_wait(tfull + 2 * grp + b, static_cast<uint32_t>((t >> 1) & 1));
            sm100::tc_fence_after();
            const uint32_t taddr = tlane + static_cast<uint32_t>(b * TILE);
            const int col_base = sq.tile() * TILE;
            if (!FOLD) {
                __syncwarp();
                reinterpret_cast<float4*>(rnw)[lane] = rn_nx;
                __syncwarp();
                UnitSeq nx = sq;
                nx.next();
                if (nx.more())
                    rn_nx = __ldg(reinterpret_cast<const float4*>(a.rnorm + nx.tile() * TILE) + lane);
            }
            auto release = [&]() {
                sm100::tc_fence_before();
                __syncwarp();
                if (lane == 0) sm100::mbar_arrive(tempty + 2 * grp + b);
            };
            if (seed) {  // seed unit: every group minimum into the 32-entry list
#pragma unroll 1
                for (int h = 0; h < 4; ++h) {
                    sm100::tmem_ld_32x32b_x32(taddr + h * 32, ra);
                    sm100::tmem_ld_wait();
                    if (h == 3) release();
                    float v[32];
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(ra[j]);
                    if (!FOLD) add_rnorm_smem(v, rnw + h * 32);
#pragma unroll
                    for (int g = 0; g < 4; ++g) {
                        const float* w = v + 8 * g;
                        const float gm = fminf(min3(min3(w[0], w[1], w[2]), min3(w[3], w[4], w[5]), w[6]), w[7]);
                        // a minimum at or above the list's last entry changes nothing
                        if (__any_sync(0xffffffffu, gm < S.key[31])) S.insert(gm);
                    }
                }
                continue;
            }
            // a unit logs <= 128 values: stop logging (the query then fails the
            // certificate and is recomputed exactly) once fewer slots are left
            tlog = ln > a.CV - 128 ? -kInf : T0;
            sm100::tmem_ld_32x32b_x32(taddr, ra);
            sm100::tmem_ld_32x32b_x32(taddr + 32, rb);
            sm100::tmem_ld_wait();
            KNN_LOG32(ra, col_base);
            sm100::tmem_ld_32x32b_x32(taddr + 64, ra);
            KNN_LOG32(rb, col_base + 32);
            sm100::tmem_ld_wait();
            sm100::tmem_ld_32x32b_x32(taddr + 96, rb);
            KNN_LOG32(ra, col_base + 64);
            sm100::tmem_ld_wait();
            release();
            KNN_LOG32(rb, col_base + 96);
        }
        if (cur_p >= 0) finish();
#undef KNN_LOG32
    }

    sm100::pdl_trigger();
    sm100::tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        sm100::tc_fence_after();
        sm100::tmem_dealloc(tmem, 512);
    }
}

}  // namespace

void launch_filter(int Kq, const CUtensorMap& tq, const CUtensorMap& tr, const CUtensorMap& tqt,
                   const CUtensorMap& trt, const FilterArgs& fa, int G, size_t smem, cudaStream_t stream) {
    auto go = [&](auto kern) {
        KNN_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            static_cast<int>(smem)));
        ProfileScope ps(stream, "tc_filter_kernel");
        KNN_CUDA_CHECK(launch_kernel(kern, G, THREADS, smem, stream, pdl_enabled(1), tq, tr, tqt, trt, fa));
    };
#define KNN_F(KRV) \
    if (fa.fold) go(filter_kernel<KRV, true>); else go(filter_kernel<KRV, false>)
    switch (Kq) {
        case 4: KNN_F(4); break;
        case 8: KNN_F(8); break;
        case 12: KNN_F(12); break;
        case 16: KNN_F(16); break;
        case 20: KNN_F(20); break;
        case 24: KNN_F(24); break;
        default: KNN_F(32); break;
    }
#undef KNN_F
    KNN_LAUNCH_CHECK();
}

void launch_filter_fixed(const CUtensorMap& tq, const CUtensorMap& tr, const CUtensorMap& tqt,
                         const CUtensorMap& trt, const FilterArgs& fa, int G, size_t smem,
                         cudaStream_t stream) {
    auto kern = fa.fold ? filter_fixed_kernel<true> : filter_fixed_kernel<false>;
    KNN_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(smem)));
    {
        ProfileScope ps(stream, "tc_filter_fixed_kernel");
        KNN_CUDA_CHECK(launch_kernel(kern, G, THREADS, smem, stream, pdl_enabled(1), tq, tr, tqt, trt, fa));
    }
    KNN_LAUNCH_CHECK();
}

}  // namespace tp
}  // namespace knnb200
