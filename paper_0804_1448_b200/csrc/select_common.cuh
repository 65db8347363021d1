// select_common.cuh -- block-wide selection building blocks shared by the
// large-k selections of the tensor path (tensor_select.cu) and of the exact
// path (exact_large.cu): bitonic sort of (key, index) pairs, radix select of
// the k-th smallest key, block prefix sums.
#pragma once

#include <cstdint>

#include "common.cuh"

namespace knnb200 {
namespace sel {

// ordered-uint encoding of floats (radix digits follow the float order)
__device__ __forceinline__ unsigned ord(float f) {
    const unsigned u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float unord(unsigned u) {
    return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}

namespace {

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
    if (active) {
#pragma unroll
        for (int j = 0; j < E; ++j) {
            rk[j] = key[t * E + j];
            ri[j] = idx[t * E + j];
        }
    }
    for (int size = 2; size <= N; size <<= 1) {
        int stride = size >> 1;
        if (stride >= W) {  // cross-warp strides (nthreads > 32 only)
            __syncthreads();  // everyone is done reading the previous shared phase
            if (active) {
#pragma unroll
                for (int j = 0; j < E; ++j) {
                    key[t * E + j] = rk[j];
                    idx[t * E + j] = ri[j];
                }
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
            if (active) {
#pragma unroll
                for (int j = 0; j < E; ++j) {
                    rk[j] = key[t * E + j];
                    ri[j] = idx[t * E + j];
                }
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
    if (active) {
#pragma unroll
        for (int j = 0; j < E; ++j) {
            key[t * E + j] = rk[j];
            idx[t * E + j] = ri[j];
        }
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
// on ord() bits, most significant digit first.  hist: 256 shared counters.
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
                const unsigned u = ord(x[e]);
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
    return unord(prefix);
}

// Block-wide exclusive prefix sum of one int per thread (NT threads); the
// block total in *total.  Contains barriers: every thread must call it.
template <int NT>
__device__ int block_exclusive_scan(int v, int* total) {
    __shared__ int s_w[NT / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    __syncthreads();  // s_w of a previous call has been read
    if (lane == 31) s_w[w] = incl;
    __syncthreads();
    int base = incl - v, tot = 0;
#pragma unroll
    for (int x = 0; x < NT / 32; ++x) {
        base += x < w ? s_w[x] : 0;
        tot += s_w[x];
    }
    *total = tot;
    return base;
}

// An upper bound B >= the k-th smallest of x[0..n) (at least k finite values;
// +inf entries are ignored)
// from ONE histogram pass: 256 linear bins over [min, hi]; B = the largest
// value in the bins up to the one where the running count reaches k, so at
// least k values are <= B (a valid bound, at most one bin above the exact
// k-th).  hist: 256 shared counters; red: 2 shared words.
__device__ float block_kth_upper_bound(const float* x, int n, int k, float hi, unsigned* hist, unsigned* red) {
    const int t = threadIdx.x;
    for (int b = t; b < 256; b += blockDim.x) hist[b] = 0u;
    __shared__ unsigned s_hi;
    if (t == 0) {
        red[0] = 0xffffffffu;  // min (ordered bits)
        red[1] = 0u;           // result (ordered bits)
        s_hi = 0u;             // max finite value (ordered bits)
    }
    __syncthreads();
    // the bins span the finite values only (a log may hold +inf padding
    // references when its threshold is infinite; they never count)
    unsigned lo_l = 0xffffffffu, hi_l = 0u;
    for (int e = t; e < n; e += blockDim.x) {
        const float v = x[e];
        if (v < kInf) {
            lo_l = min(lo_l, ord(v));
            hi_l = max(hi_l, ord(v));
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        lo_l = min(lo_l, __shfl_xor_sync(0xffffffffu, lo_l, o));
        hi_l = max(hi_l, __shfl_xor_sync(0xffffffffu, hi_l, o));
    }
    if ((t & 31) == 0) {
        atomicMin(red, lo_l);
        atomicMax(&s_hi, hi_l);
    }
    __syncthreads();
    const float lo = unord(red[0]);
    const float hi_f = fminf(hi, unord(s_hi));
    const float scale = hi_f > lo ? 256.f / (hi_f - lo) : 0.f;
    auto bin_of = [&](float v) { return min(255, max(0, static_cast<int>((v - lo) * scale))); };
    for (int e = t; e < n; e += blockDim.x)
        if (x[e] < kInf) atomicAdd(hist + bin_of(x[e]), 1u);
    __syncthreads();
    __shared__ int s_bin;
    if (t < 32) {  // warp 0: the bin where the running count reaches k
        unsigned c[8], tot = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            c[j] = hist[8 * t + j];
            tot += c[j];
        }
        unsigned incl = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
            if (t >= o) incl += y;
        }
        const unsigned excl = incl - tot;
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
    unsigned mx = 0u;
    for (int e = t; e < n; e += blockDim.x)
        if (x[e] < kInf && bin_of(x[e]) <= bk) mx = max(mx, ord(x[e]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((t & 31) == 0) atomicMax(red + 1, mx);
    __syncthreads();
    return unord(red[1]);
}

// The k smallest of n (key, index) pairs in (key, index) order by a bucket
// sort: nb (power of two) linear bins over [min, max] of the keys (bin_of is
// monotone in the key, so bin order is key order), a count pass, a prefix
// sum, a scatter of the entries of the bins up to the one where the count
// reaches k, and each entry placed by its rank among its bin's few entries.
// O(n) work and seven barriers where the bitonic network needs n log^2 n and
// dozens.  On success key/idx[0..k) hold the result (ok / oi: scratch for
// the scattered bins) and it returns true; it returns false (key / idx
// untouched) when the keys do not spread -- a bin up to the k-th holding
// more than 32 entries (dense ties), equal or non-finite extremes -- and the
// caller sorts instead.  cnt: nb shared counters (16-byte aligned); red: 3
// shared words.
template <int NT>
__device__ bool block_bucket_topk(float* key, int* idx, int n, int k, float* ok, int* oi,
                                  unsigned* cnt, int nb, unsigned* red) {
    const int t = threadIdx.x;
    for (int b = t; b < nb; b += NT) cnt[b] = 0u;
    if (t == 0) {
        red[0] = 0xffffffffu;  // min (ordered bits)
        red[1] = 0u;           // max (ordered bits)
        red[2] = 0u;           // [bk << 1 | dense]
    }
    unsigned lo_l = 0xffffffffu, hi_l = 0u;
    for (int e = t; e < n; e += NT) {
        const unsigned u = ord(key[e]);
        lo_l = min(lo_l, u);
        hi_l = max(hi_l, u);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        lo_l = min(lo_l, __shfl_xor_sync(0xffffffffu, lo_l, o));
        hi_l = max(hi_l, __shfl_xor_sync(0xffffffffu, hi_l, o));
    }
    __syncthreads();  // red / cnt initialised
    if ((t & 31) == 0) {
        atomicMin(red, lo_l);
        atomicMax(red + 1, hi_l);
    }
    __syncthreads();
    const float lo = unord(red[0]), hi = unord(red[1]);
    const float scale = static_cast<float>(nb) / (hi - lo);
    if (!(hi > lo) || !(scale < kInf) || !(hi < kInf)) return false;  // block-uniform
    auto bin_of = [&](float v) { return min(nb - 1, static_cast<int>((v - lo) * scale)); };
    for (int e = t; e < n; e += NT) atomicAdd(cnt + bin_of(key[e]), 1u);
    __syncthreads();
    // counts -> starts; thread t owns bins [t per, t per + per), read and
    // written as 16-byte vectors when per >= 4 (cnt 16-byte aligned): scalar
    // accesses at stride per would conflict per-way on the banks
    const int per = (nb + NT - 1) / NT;
    const int b0 = min(nb, t * per), b1 = min(nb, b0 + per);
    unsigned flag = 0u;
    int total = 0;
    if (per == 4 || per == 8) {  // nb = per NT: b1 - b0 == per
        uint4 c4[2];
        int own = 0;
#pragma unroll
        for (int h = 0; h < 2; ++h)
            if (4 * h < per) {
                c4[h] = *reinterpret_cast<const uint4*>(cnt + b0 + 4 * h);
                own += static_cast<int>(c4[h].x + c4[h].y + c4[h].z + c4[h].w);
            }
        int run = block_exclusive_scan<NT>(own, &total);
#pragma unroll
        for (int h = 0; h < 2; ++h)
            if (4 * h < per) {
                unsigned c[4] = {c4[h].x, c4[h].y, c4[h].z, c4[h].w};
                unsigned st[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int cj = static_cast<int>(c[j]);
                    if (run < k && cj > 32) flag = 1u;
                    if (run < k && k <= run + cj) flag |= static_cast<unsigned>(b0 + 4 * h + j) << 1;
                    st[j] = static_cast<unsigned>(run);
                    run += cj;
                }
                *reinterpret_cast<uint4*>(cnt + b0 + 4 * h) = make_uint4(st[0], st[1], st[2], st[3]);
            }
    } else {
        int own = 0;
        for (int b = b0; b < b1; ++b) own += static_cast<int>(cnt[b]);
        int run = block_exclusive_scan<NT>(own, &total);
        for (int b = b0; b < b1; ++b) {
            const int c = static_cast<int>(cnt[b]);
            if (run < k && c > 32) flag = 1u;
            if (run < k && k <= run + c) flag |= static_cast<unsigned>(b) << 1;
            cnt[b] = static_cast<unsigned>(run);
            run += c;
        }
    }
    if (flag) atomicOr(red + 2, flag);
    __syncthreads();
    const unsigned rf = red[2];
    if (rf & 1u) return false;
    const int bk = static_cast<int>(rf >> 1);
    for (int e = t; e < n; e += NT) {
        const float v = key[e];
        const int b = bin_of(v);
        if (b <= bk) {
            const unsigned pos = atomicAdd(cnt + b, 1u);
            ok[pos] = v;
            oi[pos] = idx[e];
        }
    }
    __syncthreads();  // cnt[b] = end of bin b; key / idx are free
    // final places: an entry's rank inside its bin (<= 32 entries) under the
    // (key, index) order, one thread per entry
    const int nout = static_cast<int>(cnt[bk]);
    for (int x = t; x < nout; x += NT) {
        const float kx = ok[x];
        const int ix = oi[x];
        const int b = bin_of(kx);
        const int s0 = b > 0 ? static_cast<int>(cnt[b - 1]) : 0, s1 = static_cast<int>(cnt[b]);
        int r = s0;
        for (int y = s0; y < s1; ++y) r += pair_less(ok[y], oi[y], kx, ix) ? 1 : 0;
        key[r] = kx;
        idx[r] = ix;
    }
    __syncthreads();
    return true;
}

}  // namespace

}  // namespace sel
}  // namespace knnb200
