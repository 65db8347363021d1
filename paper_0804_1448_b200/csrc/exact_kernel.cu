// exact_kernel.cu -- exact FP32 SIMT distance tiles with fused top-k.
//
// Replaces the reference's hot loops (paths relative to /root/reference/proj):
//   HOT LOOP #1  fill_key_row -> euclidean_key / manhattan_key / chebyshev_key
//                (src/bruteforce.cpp:23-38, include/knn/metric.hpp:22-44)
//   HOT LOOP #2  select_k_smallest (src/topk.cpp:17-33)
// The reference materialises a chunk x m row of double keys and selects per
// row.  Here a CTA owns 128 queries, streams 128-reference tiles through a
// cp.async shared-memory pipeline, computes the 128x128 key tile in registers
// (8x8 per thread, packed FP32 pairs, coordinates in the reference's fixed
// order), and offers each query's keys that beat its running threshold to a
// warp-cooperative sorted top-k list (warp_list.cuh) straight from registers.
// The n x m key matrix never reaches HBM.
//
// This is the engine's exact path: all metrics, any k, any d.  It is also the
// certification fallback of the tensor path (tensor_kernel.cu) and the
// re-rank arithmetic reference (key_step<M> in common.cuh).
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "exact_kernel.cuh"
#include "profile.cuh"
#include "sm100.cuh"
#include "warp_list.cuh"

namespace knnb200 {

namespace {

// CTA tile: 128 queries x 128 references, 256 threads, 8 x 8 keys per thread
// (rows ty + 16 i, reference pairs tx + 16 jp).  Coordinates stream through a
// two-stage cp.async pipeline in 32-coordinate chunks:
//   Q stage  [128 rows][QP]        row-major (reads are 2-address broadcasts)
//   R stage  [64 pairs][RPS]       two references interleaved per coordinate:
//                                  r0c0 r1c0 r0c1 r1c1 ...  so one 16-byte
//                                  load yields the packed pairs (r0,r1) at c
//                                  and c+1 -- the operand shape of the sm_100
//                                  packed FADD2/FFMA2 (fma.rn.f32x2) with the
//                                  query coordinate as the broadcast scalar.
// Every key is still accumulated coordinate by coordinate in ascending order
// with round-to-nearest sub + fma (key_step<M>), so keys are bit-identical to
// the scalar formulation used by the re-rank and merge paths.
constexpr int QT = 128;   // queries per CTA
constexpr int RT = 128;   // references per tile
constexpr int DC = 32;    // coordinates per stage
constexpr int QP = DC + 4;                 // Q row pitch (floats): 144 B, rows ty / ty+1 in distinct banks
constexpr int RPS = 2 * DC + 4;            // R pair pitch (floats): 272 B, 8 pairs -> 8 distinct 16 B bank groups
constexpr int QSTAGE = QT * QP;
constexpr int RSTAGE = (RT / 2) * RPS;
constexpr int STAGE = QSTAGE + RSTAGE;     // floats per pipeline stage
constexpr int NSTAGE = 2;
constexpr int THREADS = 256;
constexpr int LOADS = QT * DC / THREADS;   // 4-byte cp.async per operand per thread per stage

__device__ __forceinline__ void cp_async4(uint32_t dst, const float* src, bool valid) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(dst), "l"(src),
                 "r"(valid ? 4 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// Two key_step<M> updates at once: acc.{x,y} = key_step(acc.{x,y}, q, r.{x,y}),
// bitwise: one packed FADD2 for the differences (q broadcast, r negated by an
// operand modifier: q + (-r) == q - r exactly), then FFMA2 (L2), FADD2 with
// |t| (L1) or per-lane maxima (L-inf).
template <int M>
__device__ __forceinline__ float2 key_step2(float2 acc, float q, float2 r) {
    const float2 t = __fadd2_rn(make_float2(q, q), make_float2(-r.x, -r.y));
    if constexpr (M == kL2) {
        return __ffma2_rn(t, t, acc);
    } else if constexpr (M == kL1) {  // packed add with the |t| operand modifier
        return __fadd2_rn(acc, make_float2(fabsf(t.x), fabsf(t.y)));
    } else {  // consecutive maxima fuse into FMNMX3 (max is exact, order-free)
        return make_float2(fmaxf(acc.x, fabsf(t.x)), fmaxf(acc.y, fabsf(t.y)));
    }
}

// KP > 0: lists in shared memory, offered in register bursts of KP entries per
// lane (k <= 32 KP); KP < 0: lists in global memory, register bursts of -KP
// (128 < k <= 256); 0: lists in global memory, WarpList (k > 256; larger
// register bursts spill).
// KP == kLogKP: threshold-log mode (exact_large.cu): no lists; every key at
// or under the row's threshold t0 is appended to the segment's log.
constexpr int kLogKP = 1000;

template <int M, int KP, bool INDIRECT = false>
__global__ void __launch_bounds__(THREADS, 2) exact_knn_kernel(ExactArgs a) {
    constexpr bool LOG = KP == kLogKP;
    constexpr bool SMEM_LISTS = KP > 0 && !LOG;  // KP < 0: global lists, register bursts of -KP
    constexpr int RP = LOG ? 1 : (KP > 0 ? KP : -KP);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float* stages = reinterpret_cast<float*>(smem_raw);      // [NSTAGE][STAGE]
    float* Lk = stages + NSTAGE * STAGE;                       // [QT][k] (smem lists)
    int32_t* Li = reinterpret_cast<int32_t*>(Lk + (SMEM_LISTS ? QT * a.k : 0));
    float* sc = reinterpret_cast<float*>(Li + (SMEM_LISTS ? QT * a.k : 0)) + (threadIdx.x >> 5) * 2 * RT;
    const uint32_t stage_base = static_cast<uint32_t>(__cvta_generic_to_shared(stages));

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    const int ty = tid >> 4;   // rows ty + 16 i      (warp w: ty = 2w, 2w + 1)
    const int tx = tid & 15;   // pairs tx + 16 jp    (references 2 (tx + 16 jp) + e)
    const int half = lane >> 4;

    const int d = a.d;
    const int64_t m = a.m;
    if constexpr (LOG) {  // per-row threshold and log length in shared memory
        sc = reinterpret_cast<float*>(smem_raw) + NSTAGE * STAGE + (threadIdx.x >> 5) * 2 * RT;
        Lk = reinterpret_cast<float*>(smem_raw) + NSTAGE * STAGE + (THREADS / 32) * 2 * RT;  // [QT] thresholds
        Li = reinterpret_cast<int32_t*>(Lk + QT);                                          // [QT] log lengths
    } else if constexpr (!SMEM_LISTS) {
        Lk = a.glist_key + static_cast<size_t>(blockIdx.x) * QT * a.k;
        Li = a.glist_idx + static_cast<size_t>(blockIdx.x) * QT * a.k;
    }
    const int nchunks = (d + DC - 1) / DC;
    const int rr = 2 * (tid >> 6) + (tid & 1);
    const int rc = (tid & 63) >> 1;

    // stream-K: this CTA owns units [u, u_end) of the (query block, tile)
    // sequence; each query block it touches is one segment with its own lists
    sm100::pdl_wait();  // device fallback: the re-rank's query list is complete
    const int64_t n_eff = a.qcount ? min(a.n, static_cast<int64_t>(*a.qcount)) : a.n;
    if (n_eff <= 0) return;
    const ExactSplit sp = exact_split(n_eff, a.ntiles, gridDim.x, a.min_tiles);
    if (blockIdx.x >= sp.G) return;
    int64_t u = sp.start(blockIdx.x);
    const int64_t u_end = sp.start(blockIdx.x + 1);

    int buf = 0;
    while (u < u_end) {
        const int64_t b = u / a.ntiles;
        const int t_a = static_cast<int>(u - b * a.ntiles);
        const int t_b = static_cast<int>(min(static_cast<int64_t>(a.ntiles), t_a + (u_end - u)));
        u += t_b - t_a;
        const int64_t q0 = b * QT;
        const bool single = sp.cta_of(b * a.ntiles) == sp.cta_of((b + 1) * a.ntiles - 1);
        const size_t slot = static_cast<size_t>(blockIdx.x + b);

        // warp w owns rows 2w + h + 16 i (h < 2, i < 8): its 16 lists are private
        if constexpr (LOG) {
            if (lane < 16) {
                const int row = 2 * warp + (lane & 1) + 16 * (lane >> 1);
                const int64_t q = b * QT + row;
                // thresholds are indexed by the query's row in Q (its list row)
                const int64_t orow = q < n_eff ? (INDIRECT ? static_cast<int64_t>(a.qlist[q]) : q) : 0;
                Lk[row] = q < n_eff ? a.t0[orow * a.t0_stride] : -kInf;
                Li[row] = 0;
            }
        } else {
            for (int i = 0; i < 8; ++i)
                for (int h = 0; h < 2; ++h) {
                    const int row = 2 * warp + h + 16 * i;
                    WarpList<int32_t> L{Lk + row * a.k, Li + row * a.k, a.k};
                    L.init(lane);
                }
            __syncwarp();
            // rows past the query count (a partial last block; the few-query
            // device fallback) get a -inf threshold: never offered a key
            if (lane < 16) {
                const int row = 2 * warp + (lane & 1) + 16 * (lane >> 1);
                if (q0 + row >= n_eff) Lk[row * a.k + a.k - 1] = -kInf;
            }
        }
        __syncwarp();

        // stage loader: Q rows q0.. (row-major, 32 coords) and R rows t0..
        // (pair-interleaved).  Load s of this thread covers Q row 8 s + warp,
        // coordinate lane, and R reference t0 + 8 s + rr, coordinate rc, where a
        // warp reads 128 contiguous bytes of Q and 2 x 64 bytes of R.
        const int nq = static_cast<int>(min(static_cast<int64_t>(QT), n_eff - q0));
        auto issue = [&](int tile, int chunk, int sb) {
            const int64_t t0 = static_cast<int64_t>(tile) * RT;
            const int nr = static_cast<int>(min(static_cast<int64_t>(RT), m - t0));
            const int c0 = chunk * DC;
            const uint32_t sq = stage_base + static_cast<uint32_t>(sb * STAGE) * 4u;
            const uint32_t sr = sq + QSTAGE * 4u;
            const bool okq_c = c0 + lane < d, okr_c = c0 + rc < d;
            const float* gq = a.Q + (q0 + warp) * d + c0 + lane;
            const float* gr = a.R + (t0 + rr) * d + c0 + rc;
            uint32_t dq = sq + static_cast<uint32_t>(warp * QP + lane) * 4u;
            uint32_t dr = sr + static_cast<uint32_t>((tid >> 6) * RPS + (tid & 63)) * 4u;
#pragma unroll 1
            for (int s = 0; s < LOADS; ++s) {
                const bool okq = okq_c && 8 * s + warp < nq;
                const bool okr = okr_c && 8 * s + rr < nr;
                if constexpr (INDIRECT) {
                    const float* src = okq ? a.Q + static_cast<int64_t>(a.qlist[q0 + 8 * s + warp]) * d + c0 + lane
                                           : a.Q;
                    cp_async4(dq, src, okq);
                } else {
                    cp_async4(dq, okq ? gq : a.Q, okq);
                }
                cp_async4(dr, okr ? gr : a.R, okr);
                gq += 8 * static_cast<int64_t>(d);
                gr += 8 * static_cast<int64_t>(d);
                dq += 8 * QP * 4;
                dr += 4 * RPS * 4;
            }
            cp_async_commit();
        };

        float2 acc[8][4];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int jp = 0; jp < 4; ++jp) acc[i][jp] = make_float2(0.f, 0.f);

        // the buffer `buf` was last read two chunks ago, behind a barrier
        issue(t_a, 0, buf);
        for (int tile = t_a; tile < t_b; ++tile)
        for (int chunk = 0; chunk < nchunks; ++chunk, buf ^= 1) {
            cp_async_wait_all();
            __syncthreads();  // this stage landed for all threads; the previous one fully consumed
            if (chunk + 1 < nchunks) issue(tile, chunk + 1, buf ^ 1);
            else if (tile + 1 < t_b) issue(tile + 1, 0, buf ^ 1);

            const int c0 = chunk * DC;
            const int ng = (min(DC, d - c0) + 1) >> 1;  // coordinate pairs (a zero-filled odd tail is a no-op)
            const float* Qs = stages + buf * STAGE;
            const float* Rs = Qs + QSTAGE;
#pragma unroll 1
            for (int g = 0; g < ng; ++g) {
                float2 qv[8];
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    qv[i] = *reinterpret_cast<const float2*>(Qs + (ty + 16 * i) * QP + 2 * g);
                float2 r01[4], r23[4];  // (ref pair) at coordinates 2g and 2g + 1
#pragma unroll
                for (int jp = 0; jp < 4; ++jp) {
                    const float4 v = *reinterpret_cast<const float4*>(Rs + (tx + 16 * jp) * RPS + 4 * g);
                    r01[jp] = make_float2(v.x, v.y);
                    r23[jp] = make_float2(v.z, v.w);
                }
#pragma unroll
                for (int i = 0; i < 8; ++i)
#pragma unroll
                    for (int jp = 0; jp < 4; ++jp) {
                        acc[i][jp] = key_step2<M>(acc[i][jp], qv[i].x, r01[jp]);
                        acc[i][jp] = key_step2<M>(acc[i][jp], qv[i].y, r23[jp]);
                    }
            }

            if (chunk == nchunks - 1) {
                // tile complete: fused selection straight from registers.  Lane
                // (tx, half) holds 8 keys of row 2 warp + half + 16 i; the warp
                // votes against the rows' running thresholds (the lists' k-th
                // keys) and only offers a row pair's keys when one can enter.
                const int64_t t0 = static_cast<int64_t>(tile) * RT;
                const int64_t rem = m - t0;
                if (rem < RT) {  // partial last tile: columns past r_hi hold zero-filled keys
#pragma unroll
                    for (int jp = 0; jp < 4; ++jp) {
                        const int col = 2 * (tx + 16 * jp);
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            if (col >= rem) acc[i][jp].x = kInf;
                            if (col + 1 >= rem) acc[i][jp].y = kInf;
                        }
                    }
                }
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    float mn = fminf(acc[i][0].x, acc[i][0].y);
#pragma unroll
                    for (int jp = 1; jp < 4; ++jp) mn = fminf(mn, fminf(acc[i][jp].x, acc[i][jp].y));
                    const float thr = LOG ? Lk[2 * warp + half + 16 * i]
                                          : Lk[(2 * warp + half + 16 * i) * a.k + a.k - 1];
                    const unsigned vote = __ballot_sync(0xffffffffu, mn <= thr);
                    if (vote == 0u) continue;
                    // stage the row pair's 2 x 128 keys in the warp's scratch
                    // and offer each row 4 keys per lane (the list is loaded
                    // into registers for the burst: WarpRegList)
#pragma unroll
                    for (int jp = 0; jp < 4; ++jp)
                        *reinterpret_cast<float2*>(sc + half * RT + 2 * (tx + 16 * jp)) = acc[i][jp];
                    __syncwarp();
                    for (int h = 0; h < 2; ++h) {
                        if (((vote >> (16 * h)) & 0xffffu) == 0u) continue;
                        const int row = 2 * warp + h + 16 * i;
                        if constexpr (LOG) {
                            // append every key <= the row's threshold, column order
                            const float tr = Lk[row];
                            int c = Li[row];
                            float2* lg = a.vlog + (slot * QT + row) * static_cast<size_t>(a.CV);
#pragma unroll
                            for (int p = 0; p < 4; ++p) {
                                const int col = lane + 32 * p;
                                const float kv = sc[h * RT + col];
                                const bool ok = col < rem && kv <= tr;
                                const unsigned bal = __ballot_sync(0xffffffffu, ok);
                                const int pos = c + __popc(bal & ((1u << lane) - 1u));
                                if (ok && pos < a.CV)
                                    lg[pos] = make_float2(kv, __int_as_float(static_cast<int>(t0 + col)));
                                c += __popc(bal);
                            }
                            __syncwarp();
                            if (lane == 0) Li[row] = c;
                        } else if constexpr (RP > 0) {
                            float ck[4];
                            int32_t ci[4];
#pragma unroll
                            for (int p = 0; p < 4; ++p) {
                                const int col = lane + 32 * p;
                                const bool ok = col < rem;
                                ck[p] = ok ? sc[h * RT + col] : kInf;
                                ci[p] = ok ? static_cast<int32_t>(t0 + col) : 0x7fffffff;
                            }
                            WarpRegList<RP> L;
                            L.load(Lk + row * a.k, Li + row * a.k, a.k, lane);
                            if (L.offer<4>(ck, ci, a.k, lane)) L.store(Lk + row * a.k, Li + row * a.k, a.k, lane);
                        } else {
                            float ck[4];
                            int64_t ci[4];
#pragma unroll
                            for (int p = 0; p < 4; ++p) {
                                const int col = lane + 32 * p;
                                const bool ok = col < rem;
                                ck[p] = ok ? sc[h * RT + col] : kInf;
                                ci[p] = ok ? t0 + col : kSentinelIdx;
                            }
                            WarpList<int32_t> L{Lk + row * a.k, Li + row * a.k, a.k};
                            L.offer<4>(ck, ci, lane);
                        }
                    }
                    __syncwarp();
                }
#pragma unroll
                for (int i = 0; i < 8; ++i)
#pragma unroll
                    for (int jp = 0; jp < 4; ++jp) acc[i][jp] = make_float2(0.f, 0.f);
            }
        }
        __syncwarp();

        if constexpr (LOG) {  // the segment's log lengths (> CV: overflowed)
            __syncwarp();
            if (lane < 16) {
                const int row = 2 * warp + (lane & 1) + 16 * (lane >> 1);
                if (b * QT + row < n_eff) a.vlog_n[slot * QT + row] = Li[row];
            }
            __syncwarp();
            continue;
        }
        // emit this warp's lists: final rows when this segment is the block's
        // only one, else raw keys into the segment's slot for merge_exact
        for (int i = 0; i < 8; ++i)
            for (int h = 0; h < 2; ++h) {
                const int row = 2 * warp + h + 16 * i;
                const int64_t q = q0 + row;
                if (q >= n_eff) continue;
                float* ok_ = a.part_key + (slot * QT + row) * a.k;
                int64_t* oi_ = a.part_idx + (slot * QT + row) * a.k;
                if (single) {
                    const int64_t orow = INDIRECT ? static_cast<int64_t>(a.qlist[q]) : q;
                    ok_ = a.out_key + orow * a.k;
                    oi_ = a.out_idx + orow * a.k;
                    if (!a.raw_keys) finalize_list(Lk + row * a.k, Li + row * a.k, a.k, M, lane);
                }
                for (int t = lane; t < a.k; t += 32) {
                    const int32_t li = Li[row * a.k + t];
                    ok_[t] = Lk[row * a.k + t];
                    oi_[t] = li == 0x7fffffff ? kSentinelIdx : a.index_base + li;
                }
            }
        __syncwarp();
    }
}

size_t smem_bytes(int k, bool smem_lists) {
    const size_t stages = static_cast<size_t>(NSTAGE) * STAGE * sizeof(float);
    const size_t lists = static_cast<size_t>(QT) * k * (sizeof(float) + sizeof(int32_t));
    const size_t scratch = static_cast<size_t>(THREADS / 32) * 2 * RT * sizeof(float);
    return stages + (smem_lists ? lists : 0) + scratch;
}

// Merge of the blocks that span several CTAs: warp per query, the segment
// slots first + b .. last + b of its block (sorted raw lists), first adopted,
// the rest offered in 128-entry chunks with an early exit once a chunk's head
// fails the running threshold.  Queries of single-segment blocks are skipped
// (the exact kernel wrote them final).
constexpr int MX_WARPS = 4;

template <int M, bool SMEM_LISTS>
__global__ void __launch_bounds__(MX_WARPS * 32) merge_exact_kernel(ExactArgs a, float* gk, int64_t* gi) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int k = a.k;
    sm100::pdl_wait();  // the exact kernel's segment slots are complete
    const int64_t n_eff = a.qcount ? min(a.n, static_cast<int64_t>(*a.qcount)) : a.n;
    const ExactSplit sp = exact_split(n_eff, a.ntiles, a.max_ctas, a.min_tiles);
    for (int64_t q = static_cast<int64_t>(blockIdx.x) * MX_WARPS + warp; q < n_eff;
         q += static_cast<int64_t>(gridDim.x) * MX_WARPS) {
        const int64_t b = q / QT;
        const int row = static_cast<int>(q - b * QT);
        const int64_t first = sp.cta_of(b * a.ntiles), last = sp.cta_of((b + 1) * a.ntiles - 1);
        if (first == last) continue;
        float* lk;
        int64_t* li;
        if constexpr (SMEM_LISTS) {
            lk = reinterpret_cast<float*>(smem_raw) + warp * k;
            li = reinterpret_cast<int64_t*>(smem_raw + ((MX_WARPS * k * 4 + 15) / 16) * 16) + warp * k;
        } else {
            lk = gk + q * k;
            li = gi + q * k;
        }
        WarpList<int64_t> L{lk, li, k};
        auto part = [&](int64_t c) { return (static_cast<size_t>(c + b) * QT + row) * k; };
        for (int t = lane; t < k; t += 32) {
            lk[t] = a.part_key[part(first) + t];
            li[t] = a.part_idx[part(first) + t];
        }
        __syncwarp();
        for (int64_t c = first + 1; c <= last; ++c) {
            const float* pk = a.part_key + part(c);
            const int64_t* pi = a.part_idx + part(c);
            for (int t0 = 0; t0 < k; t0 += 128) {
                float ck[4];
                int64_t ci[4];
#pragma unroll
                for (int s = 0; s < 4; ++s) {
                    const int t = t0 + lane + 32 * s;
                    ck[s] = t < k ? pk[t] : kInf;
                    ci[s] = t < k ? pi[t] : kSentinelIdx;
                }
                float tk;
                int64_t ti;
                L.threshold(tk, ti);
                const float hk = __shfl_sync(0xffffffffu, ck[0], 0);
                const int64_t hi = __shfl_sync(0xffffffffu, ci[0], 0);
                if (!pair_less(hk, hi, tk, ti)) break;  // sorted part: the rest fails too
                L.offer<4>(ck, ci, lane);
            }
        }
        __syncwarp();
        if (!a.raw_keys) finalize_list(lk, li, k, M, lane);
        const int64_t orow = a.qlist ? static_cast<int64_t>(a.qlist[q]) : q;
        for (int t = lane; t < k; t += 32) {
            a.out_key[orow * k + t] = lk[t];
            a.out_idx[orow * k + t] = li[t];
        }
        __syncwarp();
    }
}

constexpr int kMergeSmemMaxK = 2048;

template <int M>
void launch_exact_m(const ExactArgs& a_in, cudaStream_t stream) {
    ExactArgs a = a_in;
    const bool smem_lists = a.glist_key == nullptr;
    const size_t smem = smem_bytes(a.k, smem_lists);
    a.max_ctas = exact_max_ctas(a.k, smem_lists);
    // 8 tiles per CTA at least (spreading a few-query block over fewer CTAs,
    // max(8, k / 4) tiles, measured slower for one fallback query at k = 100:
    // the merge saves 0.11 ms, the longer CTA chains cost 0.27 ms)
    a.min_tiles = 8;
    const int kp = (a.k + 31) / 32;
    // INDIRECT (query list, device-side count): the certification fallback of
    // the tensor path, small and large k
    const bool ind = a.qlist != nullptr;
    void (*kern)(ExactArgs) =
        !smem_lists ? (a.k <= 256 ? (ind ? exact_knn_kernel<M, -8, true> : exact_knn_kernel<M, -8>)
                                  : (ind ? exact_knn_kernel<M, 0, true> : exact_knn_kernel<M, 0>))
        : kp == 1   ? (ind ? exact_knn_kernel<M, 1, true> : exact_knn_kernel<M, 1>)
        : kp == 2   ? (ind ? exact_knn_kernel<M, 2, true> : exact_knn_kernel<M, 2>)
                    : (ind ? exact_knn_kernel<M, 4, true> : exact_knn_kernel<M, 4>);
    KNN_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(smem)));
    {
        ProfileScope ps(stream, smem_lists ? "exact_knn_kernel" : "exact_knn_kernel_glist");
        KNN_CUDA_CHECK(launch_kernel(kern, a.max_ctas, THREADS, smem, stream, a.qcount != nullptr && pdl_enabled(4), a));
    }
    KNN_LAUNCH_CHECK();
    // merge the blocks spread over several CTAs (host-known counts: only if any)
    if (!a.qcount) {
        const ExactSplit sp = exact_split(a.n, a.ntiles, a.max_ctas, a.min_tiles);
        const int64_t nqb = (a.n + QT - 1) / QT;
        bool any = false;
        for (int64_t b = 0; b < nqb && !any; ++b)
            any = sp.cta_of(b * a.ntiles) != sp.cta_of((b + 1) * a.ntiles - 1);
        if (!any) return;
    }
    const bool mx_smem = a.k <= kMergeSmemMaxK;
    if (!mx_smem && !a.mglist_key) throw CudaError("merge_exact: k > 2048 needs list scratch");
    const size_t mx_bytes = mx_smem ? ((MX_WARPS * static_cast<size_t>(a.k) * 4 + 15) / 16) * 16 +
                                          MX_WARPS * static_cast<size_t>(a.k) * 8
                                    : 0;
    const unsigned grid = static_cast<unsigned>(
        std::max<int64_t>(1, std::min<int64_t>((a.n + MX_WARPS - 1) / MX_WARPS, 4 * kSmCount)));
    ProfileScope ps(stream, "merge_exact_kernel");
    if (mx_smem) {
        KNN_CUDA_CHECK(cudaFuncSetAttribute(merge_exact_kernel<M, true>,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            static_cast<int>(mx_bytes)));
        KNN_CUDA_CHECK(launch_kernel(merge_exact_kernel<M, true>, grid, MX_WARPS * 32, mx_bytes, stream,
                                     pdl_enabled(4), a, static_cast<float*>(nullptr), static_cast<int64_t*>(nullptr)));
    } else {
        KNN_CUDA_CHECK(launch_kernel(merge_exact_kernel<M, false>, grid, MX_WARPS * 32, 0, stream, pdl_enabled(4),
                                     a, a.mglist_key, a.mglist_idx));
    }
    KNN_LAUNCH_CHECK();
}

}  // namespace

template <int M>
void launch_exact_log_m(const ExactArgs& a_in, cudaStream_t stream) {
    ExactArgs a = a_in;
    const size_t smem = smem_bytes(a.k, false) + 2 * QT * sizeof(float);
    a.max_ctas = exact_log_max_ctas();
    a.min_tiles = 0;  // the default split (exact_large's select re-derives it)
    auto kern = a.qlist ? exact_knn_kernel<M, kLogKP, true> : exact_knn_kernel<M, kLogKP>;
    KNN_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(smem)));
    {
        ProfileScope ps(stream, "exact_log_kernel");
        KNN_CUDA_CHECK(launch_kernel(kern, a.max_ctas, THREADS, smem, stream, false, a));
    }
    KNN_LAUNCH_CHECK();
}

int exact_log_max_ctas() {
    const size_t smem = smem_bytes(1, false) + 2 * QT * sizeof(float);
    return kSmCount * (smem <= 113 * 1024 ? 2 : 1);
}

size_t exact_smem_list_limit_k() {
    // lists in shared memory while 128 queries x k x 8 B + the stages fit 227 KB
    return 128;
}

int exact_max_ctas(int k, bool smem_lists) {
    // resident CTAs: 2 per SM while the shared-memory footprint allows it
    const size_t smem = smem_bytes(k, smem_lists);
    return kSmCount * (smem <= 113 * 1024 ? 2 : 1);  // 228 KB per SM, 1 KB reserved per CTA
}

int exact_ntiles(int64_t m) { return static_cast<int>((m + RT - 1) / RT); }

int64_t exact_slots(int64_t n, int ntiles, int max_ctas) {
    return exact_split(n, ntiles, max_ctas).G + (n + QT - 1) / QT;
}

int exact_queries_per_cta() { return QT; }

void launch_exact_log(int metric, const ExactArgs& a, cudaStream_t stream) {
    switch (metric) {
        case kL1: launch_exact_log_m<kL1>(a, stream); break;
        case kLinf: launch_exact_log_m<kLinf>(a, stream); break;
        default: launch_exact_log_m<kL2>(a, stream); break;
    }
}

void launch_exact(int metric, const ExactArgs& a, cudaStream_t stream) {
    switch (metric) {
        case kL1: launch_exact_m<kL1>(a, stream); break;
        case kLinf: launch_exact_m<kLinf>(a, stream); break;
        default: launch_exact_m<kL2>(a, stream); break;
    }
}

}  // namespace knnb200
