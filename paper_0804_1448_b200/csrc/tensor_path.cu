// tensor_path.cu -- tcgen05 candidate generation + exact FP32 re-rank (L2).
//
// Replaces the reference's distance fill + selection (paths relative to
// /root/reference/proj: src/bruteforce.cpp:23-38,81-96, include/knn/metric.hpp:22-29,
// src/topk.cpp:17-33) for the Euclidean metric with a GEMM-form filter on
// the 5th-generation tensor cores followed by an exact re-rank:
//
//  1. prep      Q, R -> centred, power-of-two-scaled fp16 copies (K-major rows,
//               K padded to 16) with the squared norm of every rounded
//               reference folded into three extra K columns (fp16 hi/mid/lo),
//               so one tcgen05.mma chain yields  A = ||r~||^2 - 2 q~.r~  directly.
//               Per point it also records delta = ||x~ - (x-mu)s|| (the
//               rounding radius) for the certificate.
//  2. filter    persistent, warp-specialised kernel: TMA producer warp,
//               single-thread MMA issuer (M=128 queries x N=128 references x
//               K, fp32 accumulators in 4 TMEM buffers), 8 epilogue warps
//               (thread = query row of the 32x32b TMEM load) that scan the
//               accumulators with FMNMX3 group minima against a per-query
//               running threshold and keep a sorted candidate list of the
//               K' = k+8 smallest A.  Work is split stream-K style so every
//               SM gets the same number of 128x128 tiles.
//  3. re-rank   warp per query: merge the candidate lists, derive the rigorous
//               inclusion bound tau from the k-th smallest A,
//               recompute the exact FP32 key of every candidate with A <= tau
//               (key_step<kL2>, bitwise the exact kernel's arithmetic) and keep
//               the exact top-k under the (key, index) order.
//  4. fallback  queries whose certificate fails (a candidate list overflowed
//               inside the bound: heavy near-ties/duplicates) are recomputed by
//               the exact SIMT kernel.  Results are therefore bitwise identical
//               to the exact path.
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
#include "sm100.cuh"
#include "tensor_path.cuh"
#include "tmap.cuh"
#include "warp_list.cuh"

namespace knnb200 {

namespace {

constexpr int TILE = 128;          // queries per MMA tile (M) and references per tile (N)
constexpr int EPI_WARPS = 8;       // two sets of four (one warp per TMEM lane quarter)
constexpr int EPI_THREADS = EPI_WARPS * 32;
constexpr int THREADS = 128 + EPI_THREADS;  // producer, MMA, TMEM-alloc, spare + epilogue
constexpr int KEXTRA = 0;          // bound list K' >= k + KEXTRA
constexpr int kLogGroups = 256;    // minimum logged candidate groups per (query, CTA part)
constexpr int kMaxLargeK = 1024;   // k > MAX_KQ: fixed-threshold filter + block selection
constexpr int MAX_KQ = 32;
constexpr int SMEM_LIMIT = 232448; // 227 KB opt-in per CTA

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

// Per-dimension min / max over the rows of X (both point sets).  Grid-stride
// over rows with a fixed column group per thread (VEC columns, 16-B loads when
// d % 4 == 0), so loads are coalesced and independent; the block reduces in
// shared memory and issues one global atomic per column.
template <int VEC>
__global__ void __launch_bounds__(256) range_kernel(const float* X, int64_t rows, int d, unsigned* mn,
                                                    unsigned* mx) {
    __shared__ unsigned smn[128], smx[128];
    for (int c = threadIdx.x; c < d; c += blockDim.x) {
        smn[c] = 0xffffffffu;
        smx[c] = 0u;
    }
    __syncthreads();
    const int dq = d / VEC;                       // column groups per row
    const int rpb = static_cast<int>(blockDim.x) / dq;  // rows per block step
    const int t = threadIdx.x;
    if (t < rpb * dq) {
        const int cg = t % dq, rs = t / dq;
        float lo[VEC], hi[VEC];
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
            lo[v] = kInf;
            hi[v] = -kInf;
        }
        const int64_t step = static_cast<int64_t>(gridDim.x) * rpb;
#pragma unroll 4
        for (int64_t r = static_cast<int64_t>(blockIdx.x) * rpb + rs; r < rows; r += step) {
            if constexpr (VEC == 4) {
                const float4 x4 = __ldg(reinterpret_cast<const float4*>(X + r * d) + cg);
                const float x[4] = {x4.x, x4.y, x4.z, x4.w};
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    lo[v] = fminf(lo[v], x[v]);
                    hi[v] = fmaxf(hi[v], x[v]);
                }
            } else {
                const float x = __ldg(X + r * d + cg);
                lo[0] = fminf(lo[0], x);
                hi[0] = fmaxf(hi[0], x);
            }
        }
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
            if (lo[v] <= hi[v]) {
                atomicMin(smn + cg * VEC + v, enc(lo[v]));
                atomicMax(smx + cg * VEC + v, enc(hi[v]));
            }
        }
    }
    __syncthreads();
    for (int c = threadIdx.x; c < d; c += blockDim.x) {
        if (smn[c] != 0xffffffffu) {
            atomicMin(mn + c, smn[c]);
            atomicMax(mx + c, smx[c]);
        }
    }
}

// centre mu_c = midrange, scale s = 2^e with max|x - mu| * s <= min(8, sqrt(30000/Kp))
__global__ void scale_kernel(const unsigned* mn, const unsigned* mx, int d, int Kp, float* mu,
                             float* scale, unsigned* gmax) {
    __shared__ float red[256];
    float m = 0.f;
    for (int c = threadIdx.x; c < d; c += blockDim.x) {
        const float lo = dec(mn[c]), hi = dec(mx[c]);
        const float mc = 0.5f * (lo + hi);
        mu[c] = mc;
        m = fmaxf(m, fmaxf(fabsf(hi - mc), fabsf(mc - lo)));
    }
    red[threadIdx.x] = m;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) red[threadIdx.x] = fmaxf(red[threadIdx.x], red[threadIdx.x + s]);
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const float M = red[0] * (1.f + 1e-5f);
        const float lim = fminf(8.f, sqrtf(30000.f / static_cast<float>(Kp)));
        float s = 1.f;
        if (M > 0.f && isfinite(M)) {
            int e;
            frexpf(lim / M, &e);  // lim/M = f * 2^e, f in [0.5, 1)
            s = ldexpf(1.f, e - 1);
        }
        *scale = s;
        gmax[0] = 0u;
        gmax[1] = 0u;
    }
}

// warp per row: fp16 conversion, folded norm, rounding radius
template <bool QUERY>
__global__ void __launch_bounds__(256) convert_kernel(PrepArgs a) {
    __shared__ float red[2][8];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const float s = *a.scale;
    if (QUERY && a.zero && blockIdx.x == 0 && threadIdx.x == 0) *a.zero = 0;
    if (QUERY && a.pair_slots)
        for (int p = static_cast<int>(blockIdx.x * blockDim.x + threadIdx.x); p < a.pairs;
             p += static_cast<int>(gridDim.x * blockDim.x)) {
            const int64_t u0 = static_cast<int64_t>(p) * a.rtiles;
            a.pair_slots[p] = first_cta_of(u0 + a.rtiles - 1, a.U, a.G) - first_cta_of(u0, a.U, a.G) + 1;
        }
    // reference sets: running maxima of the rounding radius and of ||r~||,
    // reduced per block (one global atomic per block, not per row)
    float dmax = 0.f, nmax = 0.f;
    const int64_t wstep = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
    for (int64_t row = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + wib; row < a.rows_pad;
         row += wstep) {
        const bool real = row < a.rows;
        double h2 = 0.0, e2 = 0.0;
        __half* out = a.Xh + row * a.Kp;
        float xv[5];  // this lane's coordinates, all loads in flight at once (Kp <= 160)
#pragma unroll
        for (int j = 0; j < 5; ++j) {
            const int c = lane + 32 * j;
            xv[j] = (real && c < a.d) ? __ldg(a.X + row * a.d + c) : 0.f;
        }
#pragma unroll
        for (int j = 0; j < 5; ++j) {
            const int c = lane + 32 * j;
            if (c >= a.Kp) break;
            __half h = __float2half_rn(0.f);
            if (real && c < a.d) {
                const float t = __fsub_rn(xv[j], a.mu[c]) * s;
                h = __float2half_rn(t);
                const double hv = static_cast<double>(__half2float(h));
                // fp16 rounding + the fp32 subtraction's rounding (<= 2^-24 |t|, doubled)
                const double err = fabs(hv - static_cast<double>(t)) + fabs(static_cast<double>(t)) * 0x1.0p-23;
                h2 += hv * hv;
                e2 += err * err;
                if (QUERY) h = __float2half_rn(-2.f * __half2float(h));  // exact: power-of-two scale
            }
            out[c] = h;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            h2 += __shfl_xor_sync(0xffffffffu, h2, o);
            e2 += __shfl_xor_sync(0xffffffffu, e2, o);
        }
        const float delta = static_cast<float>(sqrt(e2) * (1.0 + 0x1.0p-20)) * (1.f + 1e-6f);
        const float xn = static_cast<float>(sqrt(h2)) * (1.f + 1e-6f);
        if (lane == 0) {
            if (QUERY) {
                if (a.norm_col >= 0)
                    for (int j = 0; j < 3; ++j) out[a.norm_col + j] = __float2half_rn(1.f);
                a.qconst[row] = make_float4(static_cast<float>(h2), delta, xn, 0.f);
                if (a.tinit) a.tinit[row] = 0xffffffffu;
            } else if (a.norm_col >= 0) {
                if (real) {
                    const __half p1 = __double2half(h2);
                    const double r1 = h2 - static_cast<double>(__half2float(p1));
                    const __half p2 = __double2half(r1);
                    const double r2 = r1 - static_cast<double>(__half2float(p2));
                    out[a.norm_col] = p1;
                    out[a.norm_col + 1] = p2;
                    out[a.norm_col + 2] = __double2half(r2);
                } else {
                    out[a.norm_col] = __float2half_rn(kInf);  // padding: A = +inf
                }
            } else {
                a.norm[row] = real ? static_cast<float>(h2) : kInf;
            }
        }
        if (!QUERY && real) {
            dmax = fmaxf(dmax, delta);
            nmax = fmaxf(nmax, xn);
        }
    }
    if (!QUERY) {
        if (lane == 0) {
            red[0][wib] = dmax;
            red[1][wib] = nmax;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            float dm = 0.f, nm = 0.f;
            for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) {
                dm = fmaxf(dm, red[0][w]);
                nm = fmaxf(nm, red[1][w]);
            }
            atomicMax(a.gmax + 0, __float_as_uint(dm));  // non-negative floats order as uints
            atomicMax(a.gmax + 1, __float_as_uint(nm));
        }
    }
}

struct FilterArgs {
    int64_t n, m;
    int qtiles, rtiles;
    int pairs;             // query-tile pairs (a CTA keeps both tiles of a pair resident)
    int64_t U;             // pairs * rtiles work units (one 128-reference tile x 256 queries)
    int G;                 // CTAs
    int S_max;             // partial-list slots per query tile
    int KB;                // 64-wide K blocks
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
    float* part_A;         // [parts][Kq][128] final bound list (keys) of each part
    int* part_cnt;         // [parts][128] entries in part_A
    int* log_n;            // [parts][128] groups logged (may exceed CG: overflow)
    float4* log_v;         // [parts][128][CG][2] the 8 A values of each logged group
    int2* log_h;           // [parts][128][CG] {group minimum bits, first reference index}
    int CG;                // log capacity (groups) per (part, query)
    int drain_at;          // drain when a lane holds this many group minima (<= CAP - 16)
    int mode;              // dev only (KNN_B200_FILTER_MODE): 0 full, 2 no epilogue work, 3 no pushes
    float* sink;
    unsigned long long* stats;  // dev only (KNN_B200_FILTER_STATS)
    // large-k (filter_fixed_kernel): seed tiles per segment, per-query
    // threshold T0, compact value log {A, reference index} of capacity CV
    int W;
    int seed_off;          // 0 / 1: interleaved seed tile positions (retry uses fresh tiles)
    int seed_rank;         // T0 = thresh(seed_rank-th smallest seed group minimum)
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

constexpr int CAP = 32;        // per-lane buffered group minima awaiting the bound list (smem);
                               // drained once per tile (a tile pushes <= 16), off the TMEM path
constexpr int EPI_REGS = 232;  // setmaxnreg: epilogue warpgroups grow by what warpgroup 0 frees
// (the pool is the CTA's launch allocation: 2 x 128 x (232 - 168) = 128 x (168 - 40))
constexpr int CTRL_REGS = 40;

// Predicated append of one 8-reference group (inline PTX so the predicate
// never becomes a branch): if gm <= tf, the group minimum goes to the lane's
// smem buffer (bound-list input, drained later) and, while the query's log
// has room (room != 0), the 8 A values and the group's first reference index
// go to the global group log (the re-rank's candidate source).
__device__ __forceinline__ void push_group(float gm, float tf, uint32_t sg, int room, float4* lv,
                                           int2* lh, const float* w, int col) {
    asm volatile(
        "{\n\t.reg .pred p, q;\n\t"
        "setp.le.f32 p, %0, %1;\n\t"
        "setp.ne.and.s32 q, %3, 0, p;\n\t"
        "@p st.shared.f32 [%2], %0;\n\t"
        "@q st.global.v4.f32 [%4], {%6, %7, %8, %9};\n\t"
        "@q st.global.v4.f32 [%4+16], {%10, %11, %12, %13};\n\t"
        "@q st.global.v2.b32 [%5], {%0, %14};\n\t}" ::"f"(gm),
        "f"(tf), "r"(sg), "r"(room), "l"(lv), "l"(lh), "f"(w[0]), "f"(w[1]), "f"(w[2]), "f"(w[3]),
        "f"(w[4]), "f"(w[5]), "f"(w[6]), "f"(w[7]), "r"(col)
        : "memory");
}

// push_group with the bookkeeping folded into the predicates: `off` counts the
// groups logged by this (query, part) including overflow (slot = off), `sgp`
// is the next smem buffer slot; both advance only on a hit.
template <int STRIDE>
__device__ __forceinline__ void push_group_off(float gm, float tf, uint32_t& sgp, int& off, int cg,
                                               const float4* lvb, const int2* lhb, const float* w,
                                               int col) {
    asm volatile(
        "{\n\t.reg .pred p, q;\n\t.reg .u64 a, b;\n\t"
        "setp.le.f32 p, %2, %3;\n\t"
        "setp.lt.and.s32 q, %1, %4, p;\n\t"
        "@p st.shared.f32 [%0], %2;\n\t"
        "mad.wide.s32 a, %1, 32, %5;\n\t"
        "mad.wide.s32 b, %1, 8, %6;\n\t"
        "@q st.global.v8.f32 [a], {%8, %9, %10, %11, %12, %13, %14, %15};\n\t"
        "@q st.global.v2.b32 [b], {%2, %7};\n\t"
        "@p add.s32 %1, %1, 1;\n\t"
        "@p add.s32 %0, %0, %16;\n\t}"
        : "+r"(sgp), "+r"(off)
        : "f"(gm), "f"(tf), "r"(cg), "l"(lvb), "l"(lhb), "r"(col), "f"(w[0]), "f"(w[1]), "f"(w[2]),
          "f"(w[3]), "f"(w[4]), "f"(w[5]), "f"(w[6]), "f"(w[7]), "n"(STRIDE)
        : "memory");
}

// no-fold layouts: add ||r~||^2 of 32 consecutive references to the raw -2 q~.r~
__device__ __forceinline__ void add_rnorm(float (&v)[32], const float* rn) {
    const float4* nr = reinterpret_cast<const float4*>(rn);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const float4 w = __ldg(nr + j);
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
                                              const FilterArgs& a, const Pipe& P, int64_t ub,
                                              int64_t ue, int W) {
    sm100::tma_prefetch(tq);
    sm100::tma_prefetch(tr);
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
            for (int g = 0; g < 2; ++g)
                for (int kb = 0; kb < a.KB; ++kb)
                    sm100::tma_load_2d(P.As + g * P.KBB + kb * 16384, tq, P.a_full, kb * 64,
                                       (2 * sq.p + g) * TILE);
            cur_p = sq.p;
        }
        sm100::mbar_wait_sleep(P.empty + stage, phase ^ 1u);
        sm100::mbar_expect_tx(P.full + stage, static_cast<uint32_t>(P.KBB));
        unsigned char* dst = P.Bs + stage * P.KBB;
        const int rt = sq.tile();
        for (int kb = 0; kb < a.KB; ++kb)
            sm100::tma_load_2d(dst + kb * 16384, tr, P.full + stage, kb * 64, rt * TILE);
        if (++stage == a.stages) {
            stage = 0;
            phase ^= 1u;
        }
    }
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
            sm100::mbar_wait(P.a_full, a_par);
            a_par ^= 1u;
            cur_p = sq.p;
        }
        const int b = static_cast<int>(t & 1);
        const uint32_t tpar = static_cast<uint32_t>((t >> 1) & 1);
        sm100::mbar_wait(P.full + stage, phase);
        sm100::tc_fence_after();
        const uint32_t b0 = sm100::smem_u32(P.Bs + stage * P.KBB);
        {
            sm100::mbar_wait(P.tempty + 2 * g + b, tpar ^ 1u);
            sm100::tc_fence_after();
            const uint32_t a0 = sm100::smem_u32(P.As + g * P.KBB);
            const uint32_t dt = P.tmem + static_cast<uint32_t>((2 * g + b) * TILE);
            for (int ks = 0; ks < a.nslices; ++ks) {
                const uint32_t off = static_cast<uint32_t>((ks >> 2) * 16384 + (ks & 3) * 32);
                sm100::mma_f16_ss(dt, sm100::sdesc_k_sw128(a0 + off), sm100::sdesc_k_sw128(b0 + off),
                                  idesc, ks > 0 ? 1u : 0u);
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
template <int KR>
__global__ void __launch_bounds__(THREADS, 1)
    filter_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tr,
                  FilterArgs a) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1024-B aligned start, derived by offset so the compiler keeps the shared
    // address space (LDS/STS instead of generic accesses)
    unsigned char* base = smem_raw + ((1024u - (sm100::smem_u32(smem_raw) & 1023u)) & 1023u);
    const int KBB = a.KB * 16384;  // bytes of one 128-row operand tile
    unsigned char* As = base;                // 2 query tiles
    unsigned char* Bs = base + 2 * KBB;      // stages x reference tile
    float* GB = reinterpret_cast<float*>(Bs + a.stages * KBB);        // [CAP][512] group minima
    uint64_t* sT = reinterpret_cast<uint64_t*>(GB + CAP * EPI_THREADS);  // [2][128] tagged bounds
    uint64_t* sP = sT + 2 * TILE;                                       // [2][2][128] tagged kp-th
    uint64_t* bars = sP + 4 * TILE;
    uint64_t* full = bars;
    uint64_t* empty = bars + a.stages;
    uint64_t* a_full = bars + 2 * a.stages;
    uint64_t* a_empty = a_full + 1;
    uint64_t* tfull = a_full + 2;  // [query tile][parity]
    uint64_t* tempty = tfull + 4;  // [query tile][parity]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 4);

    const int warp = threadIdx.x >> 5;
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
    for (int i = threadIdx.x; i < 6 * TILE; i += blockDim.x) sT[i] = ~0ull;  // no tag matches
    if (warp == 2) sm100::tmem_alloc(tmem_slot, 512);
    sm100::tc_fence_before();
    __syncthreads();
    sm100::tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp < 4) sm100::reg_dealloc<CTRL_REGS>();
    const Pipe P{As, Bs, KBB, full, empty, a_full, a_empty, tfull, tempty, tmem};
    if (warp == 0) {
        if (sm100::elect_one()) producer_role(&tq, &tr, a, P, u_begin, u_end, 0);
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
        float T = kInf;    // own bound: thresh(k-th smallest group minimum of this list)
        float Tf = kInf;   // filter bound: min over every valid bound for this query
        unsigned tg_pref = 0xffffffffu;  // prefetched cross-CTA bound (ordered uint)
        Consts qc{};
        int64_t q = 0;
        int64_t part = 0;
        const float4* lvb = nullptr;  // this (query, part)'s group log
        const int2* lhb = nullptr;
        int ln = 0;            // groups logged so far (may exceed CG: overflow)
        unsigned long long st_drains = 0, st_rounds = 0;
        long long st_cyc_drain = 0, st_cyc_wait = 0;
        const long long st_cyc0 = kStats ? clock64() : 0;

        // Drain: one buffered group minimum per lane per round into the bound
        // list, then refresh the bound from (1) this list, (2) the other
        // parity's list of the same query (smem, tagged by pair), (3) the union
        // of both lists' ceil(k/2)-th values, (4) other CTAs' lists (global
        // atomicMin, read one drain late so the load latency hides).
#define KNN_DRAIN()                                                                              \
    do {                                                                                         \
        const long long c0_ = (kStats && a.stats) ? clock64() : 0;                                           \
        if (kStats && a.stats) ++st_drains;                                                                \
        const int nb = static_cast<int>((sgp - sg0) / (EPI_THREADS * 4));                       \
        const int mx_ = __reduce_max_sync(0xffffffffu, nb);                                      \
        _Pragma("unroll 1") for (int j_ = 0; j_ < mx_; ++j_) {                                   \
            if (kStats && a.stats) ++st_rounds;                                                            \
            const float g_ = j_ < nb ? lds_f32(sg0 + j_ * (EPI_THREADS * 4)) : kInf;             \
            /* a minimum at or above the list's last entry changes nothing */                  \
            if (__any_sync(0xffffffffu, g_ <= Tf && g_ < L.key[KR - 1])) L.insert(g_);           \
        }                                                                                        \
        sgp = sg0;                                                                               \
        if (L.cnt >= k) T = fminf(T, thresh(L.kth(k), qc));                                      \
        float tf_ = fminf(T, dec_or_inf(tg_pref));                                               \
        if (T < kInf) atomicMin(a.tglob + q, enc(T));                                            \
        tg_pref = __ldcg(a.tglob + q);                                                           \
        Tf = tf_;                                                                                \
        if (kStats && a.stats) st_cyc_drain += clock64() - c0_;                                            \
    } while (0)

#define KNN_FLUSH()                                                                              \
    do {                                                                                         \
        float* pa_ = a.part_A + part * a.Kq * TILE;                                              \
        _Pragma("unroll") for (int e_ = 0; e_ < KR; ++e_)                                        \
            if (e_ < L.cnt) pa_[e_ * TILE + row] = L.key[e_];                                    \
        a.part_cnt[part * TILE + row] = L.cnt;                                                   \
        a.log_n[part * TILE + row] = ln;                                                         \
    } while (0)

        // One 32-column chunk, branch-free: the minimum of each 8-column group
        // (FMNMX3); every group whose minimum is under the lane's bound is
        // pushed (predicated stores): its minimum to the smem buffer, its 8
        // values to the global log.  With 32 queries per warp some lane hits
        // in most chunks, so a hit must not cost a divergent branch.
#define KNN_SCAN_CHUNK(vv, colb)                                                                 \
    do {                                                                                         \
        float gm_[4];                                                                            \
        bool any_ = false;                                                                       \
        _Pragma("unroll") for (int i_ = 0; i_ < 4; ++i_) {                                       \
            const float* w_ = vv + 8 * i_;                                                       \
            gm_[i_] = fminf(min3(min3(w_[0], w_[1], w_[2]), min3(w_[3], w_[4], w_[5]), w_[6]),   \
                            w_[7]);                                                              \
            any_ |= gm_[i_] <= Tf;                                                               \
        }                                                                                        \
        if (a.mode != 3 && __any_sync(0xffffffffu, any_)) { /* some lane pushes: most chunks */ \
            _Pragma("unroll") for (int i_ = 0; i_ < 4; ++i_)                                     \
                push_group_off<EPI_THREADS * 4>(gm_[i_], Tf, sgp, ln, a.CG, lvb, lhb, vv + 8 * i_, \
                                                (colb) + 8 * i_);                                \
        }                                                                                        \
    } while (0)

        int p = static_cast<int>(u_begin / a.rtiles);
        int rt = static_cast<int>(u_begin % a.rtiles);
        const int nunits = static_cast<int>(u_end - u_begin);
        const uint32_t tlane = tmem + (static_cast<uint32_t>(quarter * 32) << 16) +
                               static_cast<uint32_t>(2 * grp * TILE);
        auto wait_full = [&](int t) {
            const long long cw_ = (kStats && a.stats) ? clock64() : 0;
            sm100::mbar_wait(tfull + 2 * grp + (t & 1), static_cast<uint32_t>((t >> 1) & 1));
            if (kStats && a.stats) st_cyc_wait += clock64() - cw_;
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
        if (a.mode != 2 && nunits > 0) {
            wait_full(0);
            sm100::tmem_ld_32x32b_x32(tlane, ra);
            sm100::tmem_ld_wait();
        }
#define KNN_SCAN_REGS(rr, colb)                                                                  \
    do {                                                                                         \
        float v_[32];                                                                            \
        _Pragma("unroll") for (int j_ = 0; j_ < 32; ++j_) v_[j_] = __uint_as_float(rr[j_]);      \
        if (!a.fold) add_rnorm(v_, a.rnorm + (colb));                                            \
        KNN_SCAN_CHUNK(v_, colb);                                                                \
    } while (0)
        for (int t = 0; t < nunits; ++t) {
            if (p != cur_p) {
                if (cur_p >= 0) {
                    KNN_DRAIN();
                    KNN_FLUSH();
                }
                cur_p = p;
                const int qt = 2 * p + grp;
                q = static_cast<int64_t>(qt) * TILE + row;
                const int slot = cta - first_cta_of(static_cast<int64_t>(p) * a.rtiles, a.U, a.G);
                part = static_cast<int64_t>(qt) * a.S_max + slot;
                const int64_t lq = (part * TILE + row) * a.CG;
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
            const int col_base = rt * TILE;
            const uint32_t taddr = tlane + static_cast<uint32_t>((t & 1) * TILE);
            if (a.mode == 2) {
                wait_full(t);
                release(t);
            } else {
                sm100::tmem_ld_32x32b_x32(taddr + 32, rb);
                KNN_SCAN_REGS(ra, col_base);
                sm100::tmem_ld_wait();
                sm100::tmem_ld_32x32b_x32(taddr + 64, ra);
                KNN_SCAN_REGS(rb, col_base + 32);
                sm100::tmem_ld_wait();
                sm100::tmem_ld_32x32b_x32(taddr + 96, rb);
                KNN_SCAN_REGS(ra, col_base + 64);
                sm100::tmem_ld_wait();
                release(t);  // all four chunks of tile t are in registers
                KNN_SCAN_REGS(rb, col_base + 96);
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
#undef KNN_SCAN_REGS
        if (cur_p >= 0) {
            KNN_DRAIN();
            KNN_FLUSH();
        }
        if (kStats && a.stats) {
            const unsigned long long lg = __reduce_add_sync(0xffffffffu, static_cast<unsigned>(ln));
            if (lane == 0) {
                atomicAdd(a.stats + 0, lg);
                atomicAdd(a.stats + 1, st_drains);
                atomicAdd(a.stats + 2, st_rounds);
                atomicAdd(a.stats + 3, lg);
                atomicAdd(a.stats + 4, static_cast<unsigned long long>(nunits));
                atomicAdd(a.stats + 5, static_cast<unsigned long long>(st_cyc_drain));
                atomicAdd(a.stats + 6, static_cast<unsigned long long>(st_cyc_wait));
                atomicAdd(a.stats + 7, static_cast<unsigned long long>(clock64() - st_cyc0));
            }
        }
#undef KNN_SCAN_CHUNK
#undef KNN_DRAIN
#undef KNN_FLUSH
    }

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
template <int DUMMY>
__global__ void __launch_bounds__(THREADS, 1)
    filter_fixed_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tr,
                        FilterArgs a) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* base = smem_raw + ((1024u - (sm100::smem_u32(smem_raw) & 1023u)) & 1023u);
    const int KBB = a.KB * 16384;
    unsigned char* As = base;
    unsigned char* Bs = base + 2 * KBB;
    uint64_t* bars = reinterpret_cast<uint64_t*>(Bs + a.stages * KBB);
    uint64_t* full = bars;
    uint64_t* empty = bars + a.stages;
    uint64_t* a_full = bars + 2 * a.stages;
    uint64_t* a_empty = a_full + 1;
    uint64_t* tfull = a_full + 2;
    uint64_t* tempty = tfull + 4;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 4);

    const int warp = threadIdx.x >> 5;
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

    if (warp < 4) sm100::reg_dealloc<CTRL_REGS>();
    const Pipe P{As, Bs, KBB, full, empty, a_full, a_empty, tfull, tempty, tmem};
    if (warp == 0) {
        if (sm100::elect_one()) producer_role(&tq, &tr, a, P, u_begin, u_end, a.W);
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
        float T0 = kInf;
        Consts qc{};
        int64_t q = 0, part = 0;
        float2* vlp = nullptr;
        int ln = 0;
        int cur_p = -1;
        bool was_seed = false;
        int64_t t = 0;
        UnitSeq sq;
        sq.init(u_begin, u_end, a.rtiles, a.W, a.seed_off);
        auto finish = [&]() {
            a.log_n[part * TILE + row] = ln;
        };
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
                if (lane < 32) a.t0[q] = T0;  // identical from every CTA of the pair
            }
            was_seed = seed;
            const int b = static_cast<int>(t & 1);
            sm100::mbar_wait(tfull + 2 * grp + b, static_cast<uint32_t>((t >> 1) & 1));
            sm100::tc_fence_after();
            const uint32_t taddr = tlane + static_cast<uint32_t>(b * TILE);
            const int col_base = sq.tile() * TILE;
#pragma unroll 1
            for (int h = 0; h < 4; ++h) {  // 32-column chunks (one TMEM load each)
                uint32_t r0[32];
                sm100::tmem_ld_32x32b_x32(taddr + h * 32, r0);
                sm100::tmem_ld_wait();
                if (h == 3) {
                    sm100::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) sm100::mbar_arrive(tempty + 2 * grp + b);
                }
                float v[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r0[j]);
                const int cb = col_base + h * 32;
                if (!a.fold) add_rnorm(v, a.rnorm + cb);
#pragma unroll
                for (int g = 0; g < 4; ++g) {
                    const float* w = v + 8 * g;
                    const float gm = fminf(min3(min3(w[0], w[1], w[2]), min3(w[3], w[4], w[5]), w[6]), w[7]);
                    if (seed) {
                        S.insert(gm);
                    } else if (__any_sync(0xffffffffu, gm <= T0)) {
                        const int col = cb + 8 * g;
                        if (ln + 8 <= a.CV) {  // room for the whole group: 3 instructions per value
                            float2* const v0 = vlp;
#pragma unroll
                            for (int e = 0; e < 8; ++e)
                                asm volatile(
                                    "{\n\t.reg .pred p;\n\t"
                                    "setp.le.f32 p, %1, %2;\n\t"
                                    "@p st.global.v2.b32 [%0], {%1, %3};\n\t"
                                    "@p add.s64 %0, %0, 8;\n\t}"
                                    : "+l"(vlp)
                                    : "f"(w[e]), "f"(T0), "r"(col + e)
                                    : "memory");
                            ln += static_cast<int>(vlp - v0);
                            continue;
                        }
#pragma unroll
                        for (int e = 0; e < 8; ++e) {
                            const int room = ln < a.CV ? 1 : 0;
                            asm volatile(
                                "{\n\t.reg .pred p, q;\n\t"
                                "setp.le.f32 p, %0, %1;\n\t"
                                "setp.ne.and.s32 q, %2, 0, p;\n\t"
                                "@q st.global.v2.b32 [%3], {%0, %4};\n\t}" ::"f"(w[e]),
                                "f"(T0), "r"(room), "l"(vlp), "r"(col + e)
                                : "memory");
                            const int hit = w[e] <= T0 ? 1 : 0;
                            vlp += hit;
                            ln += hit;
                        }
                    }
                }
            }
        }
        if (cur_p >= 0) finish();
    }

    sm100::tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        sm100::tc_fence_after();
        sm100::tmem_dealloc(tmem, 512);
    }
}

// Large-k selection, one 256-thread block per query: gather the query's
// logged {A, index} values, bitonic-sort them by A, A_(k) = k-th; certify
// (>= k logged, no overflow, thresh(A_(k)) <= T0); exact FP32 keys of every
// value <= thresh(A_(k)); bitonic sort by (key, index); top k.
constexpr int LK_THREADS = 512;
#ifndef KNN_DBG_LARGE
#define KNN_DBG_LARGE 0
#endif

// Bitonic sort of N (power of two) (key, index) pairs in shared memory under
// the (key, index) order, by `nthreads` threads (32: one warp, no block
// barriers; or the whole block).  Thread t holds elements t E .. t E + E - 1 in
// registers (E = N / nthreads): strides below E are register swaps, strides
// below 32 E are lane shuffles, and only the strides that cross warps go
// through shared memory (one barrier each) -- 18 barriers at N = 2048 where the
// all-shared-memory network needs 66.
template <int E>
__device__ void bitonic_sort_kv_regs(float* key, int* idx, int N, int nthreads) {
    const int t = threadIdx.x;
    const bool active = t < nthreads;
    const int W = 32 * E;  // elements per warp
    float rk[E];
    int ri[E];
    __syncthreads();  // the caller's writes of key/idx are visible
    if (active)
#pragma unroll
        for (int j = 0; j < E; ++j) {
            rk[j] = key[t * E + j];
            ri[j] = idx[t * E + j];
        }
    for (int size = 2; size <= N; size <<= 1) {
        int stride = size >> 1;
        if (stride >= W) {  // cross-warp strides (nthreads > 32 only)
            __syncthreads();  // everyone is done reading the previous shared phase
            if (active)
#pragma unroll
                for (int j = 0; j < E; ++j) {
                    key[t * E + j] = rk[j];
                    idx[t * E + j] = ri[j];
                }
            for (; stride >= W; stride >>= 1) {
                __syncthreads();
                for (int i = t; i < (N >> 1); i += blockDim.x) {
                    const int lo = 2 * i - (i & (stride - 1));
                    const int hi = lo + stride;
                    const bool up = (lo & size) == 0;
                    const float ka = key[lo], kb = key[hi];
                    const int ia = idx[lo], ib = idx[hi];
                    if (pair_less(kb, ib, ka, ia) == up) {
                        key[lo] = kb;
                        key[hi] = ka;
                        idx[lo] = ib;
                        idx[hi] = ia;
                    }
                }
            }
            __syncthreads();
            if (active)
#pragma unroll
                for (int j = 0; j < E; ++j) {
                    rk[j] = key[t * E + j];
                    ri[j] = idx[t * E + j];
                }
        }
        if (!active) continue;
        for (; stride >= E; stride >>= 1) {  // partner in lane ^ (stride / E), same slot
            const int lm = stride / E;
#pragma unroll
            for (int j = 0; j < E; ++j) {
                const float pk = __shfl_xor_sync(0xffffffffu, rk[j], lm);
                const int pi = __shfl_xor_sync(0xffffffffu, ri[j], lm);
                const int e = t * E + j;
                const bool keep_min = ((e & stride) == 0) == ((e & size) == 0);
                const bool p_less = pair_less(pk, pi, rk[j], ri[j]);
                if (p_less == keep_min) {
                    rk[j] = pk;
                    ri[j] = pi;
                }
            }
        }
#pragma unroll
        for (int s = E / 2; s > 0; s >>= 1) {  // partner in this thread
            if (s > stride) continue;
#pragma unroll
            for (int j = 0; j < E; ++j) {
                if (j & s) continue;
                const bool up = ((t * E + j) & size) == 0;
                if (pair_less(rk[j + s], ri[j + s], rk[j], ri[j]) == up) {
                    const float tk = rk[j];
                    const int ti = ri[j];
                    rk[j] = rk[j + s];
                    ri[j] = ri[j + s];
                    rk[j + s] = tk;
                    ri[j + s] = ti;
                }
            }
        }
    }
    __syncthreads();
    if (active)
#pragma unroll
        for (int j = 0; j < E; ++j) {
            key[t * E + j] = rk[j];
            idx[t * E + j] = ri[j];
        }
    __syncthreads();
}

// N (power of two, 32 <= N <= 16 * blockDim.x) pairs by the whole block:
// one element per thread up to N = blockDim.x, then N / blockDim.x.
__device__ void bitonic_sort_kv(float* key, int* idx, int N) {
    const int bd = static_cast<int>(blockDim.x);
    if (N <= bd) {
        bitonic_sort_kv_regs<1>(key, idx, N, N);
        return;
    }
    switch (N / bd) {
        case 2: bitonic_sort_kv_regs<2>(key, idx, N, bd); break;
        case 4: bitonic_sort_kv_regs<4>(key, idx, N, bd); break;
        case 8: bitonic_sort_kv_regs<8>(key, idx, N, bd); break;
        default: bitonic_sort_kv_regs<16>(key, idx, N, bd); break;
    }
}

// k-th smallest (1-based) of x[0..n) (finite floats), block-wide radix select
// on enc() bits, most significant digit first.  hist: 256 shared counters.
__device__ float block_kth_smallest(const float* x, int n, int k, unsigned* hist, int* scratch) {
    unsigned prefix = 0, mask = 0;
    int want = k;  // rank still to find among keys matching prefix
#pragma unroll 1
    for (int shift = 24; shift >= 0; shift -= 8) {
        for (int b = threadIdx.x; b < 256; b += blockDim.x) hist[b] = 0u;
        __syncthreads();
        // warp-aggregated increments: the leading digits of nearby keys
        // coincide, so plain atomics would serialise on one or two bins
        for (int e0 = 0; e0 < n; e0 += blockDim.x) {
            const int e = e0 + threadIdx.x;
            int bin = -1;
            if (e < n) {
                const unsigned u = enc(x[e]);
                if ((u & mask) == prefix) bin = static_cast<int>((u >> shift) & 255u);
            }
            const unsigned same = __match_any_sync(0xffffffffu, bin);
            if (bin >= 0 && (__ffs(same) - 1) == (threadIdx.x & 31))
                atomicAdd(hist + bin, static_cast<unsigned>(__popc(same)));
        }
        __syncthreads();
        if (threadIdx.x < 32) {  // warp 0: the bin holding rank `want` (8 bins per lane)
            const int l = threadIdx.x;
            unsigned c[8], tot = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                c[j] = hist[8 * l + j];
                tot += c[j];
            }
            unsigned incl = tot;  // inclusive prefix over lanes
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
                if (l >= o) incl += y;
            }
            const unsigned excl = incl - tot;
            if (excl < static_cast<unsigned>(want) && static_cast<unsigned>(want) <= incl) {
                unsigned acc = excl;
                int j = 0;
                for (; j < 7; ++j) {
                    if (acc + c[j] >= static_cast<unsigned>(want)) break;
                    acc += c[j];
                }
                scratch[0] = 8 * l + j;
                scratch[1] = want - static_cast<int>(acc);
            }
        }
        __syncthreads();
        const unsigned b = static_cast<unsigned>(scratch[0]);
        want = scratch[1];
        prefix |= b << shift;
        mask |= 255u << shift;
        __syncthreads();
    }
    return dec(prefix);
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

// NT threads per query: the fewest of 64 / 128 / 256 / 512 that hold the candidate
// capacity NC <= 16 x NT (more resident blocks, cheaper barriers)
template <int NT>
__global__ void __launch_bounds__(NT) select_large_kernel(LargeArgs a) {
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
        // A_(k) by radix select on the order-preserving key bits (4 x 8-bit
        // digits, block histograms), no sort
        const float ak = block_kth_smallest(sk, total, k, s_hist, s_sel);
        const Consts qc = load_consts(a.f, q);
        tau = thresh(ak, qc);
        ok = tau <= T0;  // every reference with A <= tau was logged
        if (ok) {
            // compact the candidates (A <= tau) to the front, any order
            if (threadIdx.x == 0) s_cnt = 0;
            __syncthreads();
            int mine[16];  // total <= NC <= 16 * NT: a thread owns <= 16 entries
            int nm = 0;
            for (int e = threadIdx.x; e < total; e += blockDim.x)
                if (sk[e] <= tau) mine[nm++] = si[e];
            __syncthreads();
            const int base = atomicAdd(&s_cnt, nm);
            for (int j = 0; j < nm; ++j) si[base + j] = mine[j];
            __syncthreads();
            nc = s_cnt;
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
    int N2 = 32;
    while (N2 < nc) N2 <<= 1;
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

// -------------------------------------------------------------- re-rank ----
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

constexpr int RR_WARPS = 4;
constexpr int RR_CAND = 128;  // exact candidates per query on the fast path (more: fallback)

__host__ __device__ constexpr size_t rr_warp_bytes(int span, int k) {
    return ((static_cast<size_t>(span) * 4 + RR_CAND * 8 + static_cast<size_t>(k) * 4 + 15) / 16) * 16 +
           static_cast<size_t>(k) * 8;
}

// Warp per query.  (1) A_bound = k-th smallest of the union of the parts'
// bound lists (rank counting over the compacted lists); tau = thresh(A_bound).
// (2) Certificate: no part's group log overflowed, so every reference with
// A <= tau is in a log (every filter bound was >= tau).  (3) Candidates =
// logged values <= tau; their exact FP32 keys (key_step<kL2>, bitwise the
// exact kernel's arithmetic); (4) exact top-k by (key, index) rank counting.
__global__ void __launch_bounds__(RR_WARPS * 32) rerank_kernel(RerankArgs a) {
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

    const int qt = static_cast<int>(q / TILE);
    const int row = static_cast<int>(q % TILE);
    const int64_t p0 = static_cast<int64_t>(qt) * parts;

    // Every step below issues its loads for the whole query at once (one
    // memory round trip per step): the kernel is latency-bound per warp.
    // part slots written for this pair: one per CTA whose unit range touches it
    const int pair = qt >> 1;
    const int nslots = a.f.pair_slots[pair];
    int cnt = 0, nlog = 0;
    if (lane < nslots) {
        cnt = a.f.part_cnt[(p0 + lane) * TILE + row];
        nlog = a.f.log_n[(p0 + lane) * TILE + row];
    }
    const Consts qc = load_consts(a.f, q);
    // 0. all bound lists, compacted: list p's entries go to [excl_p, excl_p + cnt_p)
    int cincl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, cincl, o);
        if (lane >= o) cincl += y;
    }
    const int L = __shfl_sync(0xffffffffu, cincl, 31);
    for (int p = 0; p < nslots; ++p) {  // a list holds <= Kq <= 32 entries
        const int cp = __shfl_sync(0xffffffffu, cnt, p);
        const int ep = __shfl_sync(0xffffffffu, cincl, p) - cp;
        if (lane < cp) sv[ep + lane] = a.f.part_A[((p0 + p) * Kq + lane) * TILE + row];
    }
    __syncwarp();

    // 1. k-th smallest (value, position) of the compacted lists.  Each list is
    //    sorted, so an entry's rank is its own position plus, per other list,
    //    a binary search: entries <= v of earlier lists, < v of later ones.
    float B = kInf;
    if (L >= k) {
        for (int x0 = 0; x0 < L; x0 += 32) {  // warp-uniform trip count (shuffles inside)
            const int x = x0 + lane;
            const bool valid = x < L;
            const float v = valid ? sv[x] : kInf;
            int px = 0;
            for (int p = 1; p < nslots; ++p)
                if (x >= __shfl_sync(0xffffffffu, cincl, p - 1)) px = p;
            int rank = 0;
            for (int p = 0; p < nslots; ++p) {
                const int cp = __shfl_sync(0xffffffffu, cnt, p);
                const int ep = __shfl_sync(0xffffffffu, cincl, p) - cp;
                // first entry of list p that is not "less" than (v, x)
                int lo = 0, hi = (p == px || !valid) ? 0 : cp;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    const float w = sv[ep + mid];
                    if (p < px ? w <= v : w < v) lo = mid + 1;
                    else hi = mid;
                }
                rank += p == px ? x - ep : lo;
            }
            if (valid && rank == k - 1) B = v;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) B = fminf(B, __shfl_xor_sync(0xffffffffu, B, o));
    }
    const float tau = thresh(B, qc);

    // 2. certificate
    bool ok = __all_sync(0xffffffffu, nlog <= a.f.CG) && isfinite(tau);

    // 3. candidates: logged values <= tau.  Heads of every logged group of
    //    every part (flattened over parts), then the values of the groups whose
    //    minimum is inside tau, then their values <= tau.
    int nc = 0;
    if (ok) {
        int* gl = reinterpret_cast<int*>(ck);  // in-tau groups (log slot), reuses ck
        int ng = 0;
        for (int p = 0; p < nslots; ++p) {
            const int np = __shfl_sync(0xffffffffu, nlog, p);
            const int base = static_cast<int>(((p0 + p) * TILE + row) * a.f.CG);
            for (int t0 = 0; t0 < np; t0 += 32) {
                const int t = t0 + lane;
                const bool in = t < np && __int_as_float(a.f.log_h[base + t].x) <= tau;
                const unsigned bal = __ballot_sync(0xffffffffu, in);
                const int pos = ng + __popc(bal & ((1u << lane) - 1u));
                if (in && pos < RR_CAND) gl[pos] = base + t;
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
                const int slot = gl[j];
                ldg8(reinterpret_cast<const float*>(a.f.log_v + 2 * static_cast<int64_t>(slot)), w);
                c0 = a.f.log_h[slot].y;
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

// gather / scatter for the certification fallback
__global__ void gather_rows_kernel(const float* X, int d, const int* list, int count, float* out) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t total = static_cast<int64_t>(count) * d;
    if (i >= total) return;
    const int64_t r = i / d;
    out[i] = X[static_cast<int64_t>(list[r]) * d + i % d];
}

__global__ void scatter_rows_kernel(const float* src_d, const int64_t* src_i, const int* list,
                                    int count, int k, float* out, int64_t* out_idx) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= static_cast<int64_t>(count) * k) return;
    const int64_t r = i / k;
    const int64_t dst = static_cast<int64_t>(list[r]) * k + i % k;
    out[dst] = src_d[i];
    out_idx[dst] = src_i[i];
}

struct Layout {
    int d16, Kp, KB, norm_col, stages, Kq;
    bool fold;
    size_t smem;
};

Layout layout_for(int d, int k) {
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
    const size_t epi = static_cast<size_t>(EPI_THREADS) * CAP * 4 + 6 * TILE * 8;
    const size_t fixed = epi + 1024 /*align*/ + 512 /*barriers*/;
    auto stages_for = [&](int KB) {
        const size_t per = static_cast<size_t>(KB) * 16384;
        const long avail = static_cast<long>(SMEM_LIMIT) - static_cast<long>(fixed + 2 * per);
        return avail > 0 ? static_cast<int>(avail / static_cast<long>(per)) : 0;
    };
    if (kb_fold == kb_plain || stages_for(kb_fold) >= 3) {
        L.fold = true;
        L.Kp = kfold;
        L.KB = kb_fold;
        L.norm_col = ncol;
    } else {
        L.fold = false;
        L.Kp = L.d16;
        L.KB = kb_plain;
        L.norm_col = -1;
    }
    L.stages = std::min(stages_for(L.KB), 6);
    L.smem = fixed + static_cast<size_t>(L.KB) * 16384 * (2 + L.stages);
    return L;
}

}  // namespace

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
    {
        ProfileScope ps(stream, "prep_range_kernel");
        const int vec = (d % 4 == 0) ? 4 : 1;
        const int rpb = 256 / (d / vec);
        const int64_t want = (m + rpb * 8 - 1) / (rpb * 8);  // >= 8 rows per thread
        const unsigned grid =
            static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(want, 4 * kSmCount)));
        if (vec == 4)
            range_kernel<4><<<grid, 256, 0, stream>>>(dR, m, d, mnmx, mnmx + d);
        else
            range_kernel<1><<<grid, 256, 0, stream>>>(dR, m, d, mnmx, mnmx + d);
    }
    KNN_LAUNCH_CHECK();
    {
        ProfileScope ps(stream, "prep_scale_kernel");
        scale_kernel<<<1, 256, 0, stream>>>(mnmx, mnmx + d, d, L.Kp, r.mu, r.scale, r.gmax);
    }
    KNN_LAUNCH_CHECK();
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
    {
        ProfileScope ps(stream, "prep_convert_refs");
        convert_kernel<false>
            <<<static_cast<unsigned>(std::min<int64_t>((r.m_pad + 7) / 8, 8 * kSmCount)), 256, 0,
               stream>>>(pr);
    }
    KNN_LAUNCH_CHECK();
}

void run_tensor_path(DeviceContext& ctx, cudaStream_t stream, const float* dQ, int64_t n,
                     const float* dR, int64_t m, int d, int k, int raw_keys, int64_t index_base,
                     float* d_out, int64_t* d_idx) {
    ctx.refs.reserve(tensor_refs_bytes(m, d));
    TensorRefs r;
    tensor_prep_refs(stream, dR, m, d, ctx.refs.base(), r);
    tensor_search(ctx, stream, r, dQ, n, k, raw_keys, index_base, d_out, d_idx);
}

void tensor_search(DeviceContext& ctx, cudaStream_t stream, const TensorRefs& refs,
                   const float* dQ, int64_t n, int k, int raw_keys, int64_t index_base,
                   float* d_out, int64_t* d_idx, const FallbackSink* sink, int margin, bool retry) {
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
    // at most ~29 CTAs share a query-tile pair, so a query has <= 32 partial lists
    const int G = static_cast<int>(std::min<int64_t>(std::min<int64_t>(kSmCount, U),
                                                     static_cast<int64_t>(pairs) * 29));
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
    const bool large = k > MAX_KQ;
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
    const int fb_ctas = exact_max_ctas(k, true);
    const size_t fb_part = large ? 0
                                 : static_cast<size_t>(exact_slots(n, exact_ntiles(m), fb_ctas)) *
                                       exact_queries_per_cta() * k;
    sz.take<float>(fb_part);
    sz.take<int64_t>(fb_part);
    ctx.arena.reserve(sz.used + 256);
    Carver cv{static_cast<char*>(ctx.arena.base())};
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
    {
        ProfileScope ps(stream, "prep_convert_queries");
        convert_kernel<true><<<static_cast<unsigned>(std::min<int64_t>((n_pad + 7) / 8, 8 * kSmCount)),
                               256, 0, stream>>>(pr);
    }
    KNN_LAUNCH_CHECK();

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
    auto launch_filter = [&](auto kern) {
        KNN_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            static_cast<int>(L.smem)));
        ProfileScope ps(stream, "tc_filter_kernel");
        kern<<<G, THREADS, L.smem, stream>>>(tq, tr, fa);
    };
    if (large) {
        // seed: W tiles whose 32nd smallest group minimum estimates the
        // (margin*k)-th smallest A (rank ~ m * 32 / (128 W)), W >= 2
        fa.seed_rank = 32;
        fa.W = static_cast<int>(std::min<int64_t>(
            rtiles, std::max<int64_t>(2, (m + 4LL * margin * k - 1) / (4LL * margin * k))));
        fa.seed_off = retry ? 1 : 0;
        fa.t0 = t0;
        fa.vlog = vlog;
        fa.CV = CV;
        const size_t smem_fixed = 1024 + 512 + static_cast<size_t>(L.KB) * 16384 *
                                                   (2 + std::min(L.stages + 2, 6));
        const int stages_fixed = std::min(L.stages + 2, 6);
        fa.stages = stages_fixed;
        KNN_CUDA_CHECK(cudaFuncSetAttribute(filter_fixed_kernel<0>,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            static_cast<int>(smem_fixed)));
        {
            ProfileScope ps(stream, "tc_filter_fixed_kernel");
            filter_fixed_kernel<0><<<G, THREADS, smem_fixed, stream>>>(tq, tr, fa);
        }
        KNN_LAUNCH_CHECK();
        LargeArgs la{};
        la.Q = dQ;
        la.R = dR;
        la.n = n;
        la.d = d;
        la.k = k;
        la.S_max = S_max;
        int NC = 1;
        while (NC < 2 * margin * k) NC <<= 1;
        NC = std::min(NC, 16 * LK_THREADS);
        la.NC = NC;
        la.f = fa;
        la.raw_keys = raw_keys;
        la.index_base = index_base;
        la.out = d_out;
        la.out_idx = d_idx;
        la.fb_count = sink ? sink->count : fb;
        la.fb_list = sink ? sink->list : fb + 1;
        la.fb_offset = sink ? sink->offset : 0;
        const size_t sel_smem = static_cast<size_t>(NC) * 8;
        const int nt = NC <= 16 * 64 ? 64 : NC <= 16 * 128 ? 128 : NC <= 16 * 256 ? 256 : LK_THREADS;
        auto sel = nt == 64    ? select_large_kernel<64>
                   : nt == 128 ? select_large_kernel<128>
                   : nt == 256 ? select_large_kernel<256> : select_large_kernel<LK_THREADS>;
        KNN_CUDA_CHECK(cudaFuncSetAttribute(sel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            static_cast<int>(sel_smem)));
        {
            ProfileScope ps(stream, "select_large_kernel");
            sel<<<static_cast<unsigned>(n), nt, sel_smem, stream>>>(la);
        }
        KNN_LAUNCH_CHECK();
    } else {
    switch (L.Kq) {
        case 4: launch_filter(filter_kernel<4>); break;
        case 8: launch_filter(filter_kernel<8>); break;
        case 12: launch_filter(filter_kernel<12>); break;
        case 16: launch_filter(filter_kernel<16>); break;
        case 20: launch_filter(filter_kernel<20>); break;
        case 24: launch_filter(filter_kernel<24>); break;
        default: launch_filter(filter_kernel<32>); break;
    }
    KNN_LAUNCH_CHECK();
    if (want_stats) {
        unsigned long long h[8];
        KNN_CUDA_CHECK(cudaMemcpyAsync(h, fa.stats, sizeof(h), cudaMemcpyDeviceToHost, stream));
        KNN_CUDA_CHECK(cudaStreamSynchronize(stream));
        KNN_CUDA_CHECK(cudaFree(fa.stats));
        const double warps = static_cast<double>(G) * EPI_WARPS;
        std::fprintf(stderr,
                     "[filter stats] per warp: tiles %.1f groups-pushed/lane %.1f drains %.1f insert-rounds "
                     "%.1f | logged-groups/lane %.2f | kcycles/warp: drain %.1f tfull-wait %.1f total %.1f\n",
                     h[4] / warps, h[0] / (warps * 32.0), h[1] / warps, h[2] / warps,
                     h[3] / (warps * 32.0), h[5] / warps / 1e3, h[6] / warps / 1e3, h[7] / warps / 1e3);
    }
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
    if (!large) {
        ProfileScope ps(stream, "rerank_kernel");
        rerank_kernel<<<static_cast<unsigned>((n + RR_WARPS - 1) / RR_WARPS), RR_WARPS * 32, rr_smem,
                        stream>>>(ra);
    }
    KNN_LAUNCH_CHECK();

    // 4. certification fallback (exact kernel on the failed queries), unless
    //    the caller collects them across several searches.  Small k: entirely
    //    on the device -- no host round trip, the search stays asynchronous.
    if (sink) return;
    if (!ctx.fb_dev) KNN_CUDA_CHECK(cudaMalloc(&ctx.fb_dev, sizeof(int)));
    if (!large) {
        ExactArgs ea{};
        ea.Q = dQ;
        ea.R = dR;
        ea.n = n;
        ea.m = m;
        ea.d = d;
        ea.k = k;
        ea.ntiles = exact_ntiles(m);
        ea.qlist = fb + 1;
        ea.qcount = fb;
        ea.index_base = index_base;
        ea.raw_keys = raw_keys;
        ea.out_key = d_out;
        ea.out_idx = d_idx;
        ea.part_key = fb_pk;
        ea.part_idx = fb_pi;
        launch_exact(kL2, ea, stream);
        KNN_CUDA_CHECK(cudaMemcpyAsync(ctx.fb_dev, fb, sizeof(int), cudaMemcpyDeviceToDevice, stream));
        ctx.fb_on_device = true;
        return;
    }
    ctx.fb_on_device = false;
    int fails = 0;
    KNN_CUDA_CHECK(cudaMemcpyAsync(&fails, fb, sizeof(int), cudaMemcpyDeviceToHost, stream));
    KNN_CUDA_CHECK(cudaStreamSynchronize(stream));
    if (fails > 0) {
        std::vector<int> list(static_cast<size_t>(fails));
        KNN_CUDA_CHECK(cudaMemcpy(list.data(), fb + 1, sizeof(int) * fails, cudaMemcpyDeviceToHost));
        // the fallback allocates its own scratch: keep the gathered queries in a
        // dedicated buffer so the exact path's arena use cannot clobber them
        float* gq = nullptr;
        float* od = nullptr;
        int64_t* oi = nullptr;
        int* dl = nullptr;
        KNN_CUDA_CHECK(cudaMallocAsync(&gq, sizeof(float) * fails * d, stream));
        KNN_CUDA_CHECK(cudaMallocAsync(&od, sizeof(float) * fails * k, stream));
        KNN_CUDA_CHECK(cudaMallocAsync(&oi, sizeof(int64_t) * fails * k, stream));
        KNN_CUDA_CHECK(cudaMallocAsync(&dl, sizeof(int) * fails, stream));
        KNN_CUDA_CHECK(cudaMemcpyAsync(dl, list.data(), sizeof(int) * fails, cudaMemcpyHostToDevice,
                                       stream));
        {
            const int64_t tot = static_cast<int64_t>(fails) * d;
            ProfileScope ps(stream, "fallback_gather");
            gather_rows_kernel<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, stream>>>(
                dQ, d, dl, fails, gq);
        }
        KNN_LAUNCH_CHECK();
        if (large && !retry)  // a tail estimate of T0: once more from fresh seed tiles
            tensor_search(ctx, stream, refs, gq, fails, k, raw_keys, index_base, od, oi, nullptr,
                          margin, true);
        else
            run_exact_subset(ctx, stream, gq, fails, dR, m, d, k, raw_keys, index_base, od, oi);
        {
            const int64_t tot = static_cast<int64_t>(fails) * k;
            ProfileScope ps(stream, "fallback_scatter");
            scatter_rows_kernel<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, stream>>>(
                od, oi, dl, fails, k, d_out, d_idx);
        }
        KNN_LAUNCH_CHECK();
        KNN_CUDA_CHECK(cudaFreeAsync(gq, stream));
        KNN_CUDA_CHECK(cudaFreeAsync(od, stream));
        KNN_CUDA_CHECK(cudaFreeAsync(oi, stream));
        KNN_CUDA_CHECK(cudaFreeAsync(dl, stream));
    }
    ctx.last_fallbacks = fails;
}

}  // namespace knnb200
