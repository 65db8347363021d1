// tensor_prep.cu -- tensor-path preparation of a point set: per-dimension
// range, midrange centre and power-of-two scale (reference set), then the
// fp16 copy (K-major, K padded to 16) with the folded squared norms of the
// references or the query constants, and every point's rounding radius
// (DESIGN.md sec. 3.2 step 0-1, sec. 4).
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "profile.cuh"
#include "sm100.cuh"
#include "tensor_internal.cuh"

namespace knnb200 {
namespace tp {

namespace {

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
    if (QUERY) sm100::pdl_trigger();  // the filter may start its prologue
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
        bool ovf = false;  // a query operand -2 h overflowed fp16
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
                if (QUERY) {  // exact (power-of-two scale) unless -2 h leaves the fp16 range
                    h = __float2half_rn(-2.f * __half2float(h));
                    ovf |= __hisinf(h) != 0;
                }
            }
            out[c] = h;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            h2 += __shfl_xor_sync(0xffffffffu, h2, o);
            e2 += __shfl_xor_sync(0xffffffffu, e2, o);
        }
        // an overflowed operand breaks the MMA's error model: an infinite
        // rounding radius makes every bound infinite, so the query fails the
        // certificate and is recomputed exactly
        const bool any_ovf = __any_sync(0xffffffffu, ovf);
        const float delta = any_ovf ? kInf : static_cast<float>(sqrt(e2) * (1.0 + 0x1.0p-20)) * (1.f + 1e-6f);
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

// Row-quad layout of the same conversion for d % 4 == 0 (every configuration
// of the benchmark): 4 lanes per row, 8 rows per warp.  Lane l of a row owns
// the 4-coordinate granules g = l, l + 4, ..., loads them with 128-bit loads
// (the 4 lanes of a row read 64 contiguous bytes per instruction), writes
// their fp16 images with 64-bit stores (32 contiguous bytes per row), and the
// per-row sums reduce over the 4 lanes (2 shuffle levels instead of 5).  The
// arithmetic per coordinate is convert_kernel's, so Xh, the norms and the
// radii agree with it up to the (exact-double) summation order.
#ifndef KNN_CONVERT_MINB
#define KNN_CONVERT_MINB 5  // 5 resident blocks per SM (<= 48 registers): config B's 600 blocks in one wave
#endif
template <bool QUERY, int GPL>  // GPL: granules per lane (d <= 16 GPL)
__global__ void __launch_bounds__(256, KNN_CONVERT_MINB) convert4_kernel(PrepArgs a) {
    if (QUERY) sm100::pdl_trigger();
    __shared__ float red[2][8];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int l4 = lane & 3;
    const float s = *a.scale;
    if (QUERY && a.zero && blockIdx.x == 0 && threadIdx.x == 0) *a.zero = 0;
    if (QUERY && a.pair_slots)
        for (int p = static_cast<int>(blockIdx.x * blockDim.x + threadIdx.x); p < a.pairs;
             p += static_cast<int>(gridDim.x * blockDim.x)) {
            const int64_t u0 = static_cast<int64_t>(p) * a.rtiles;
            a.pair_slots[p] = first_cta_of(u0 + a.rtiles - 1, a.U, a.G) - first_cta_of(u0, a.U, a.G) + 1;
        }
    const int ng = a.d >> 2;       // coordinate granules
    const int nk = a.Kp >> 2;      // output granules (4 halves each)
    float dmax = 0.f, nmax = 0.f;
    const int64_t rstep = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 2);
    for (int64_t row0 = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 2); row0 < a.rows_pad;
         row0 += rstep) {
        const int64_t row = row0 + (threadIdx.x >> 2);
        const bool inpad = row < a.rows_pad;
        const bool real = row < a.rows;
        float4 x[GPL];
#pragma unroll
        for (int j = 0; j < GPL; ++j) {
            const int g = 4 * j + l4;
            x[j] = (real && g < ng) ? __ldg(reinterpret_cast<const float4*>(a.X + row * a.d) + g)
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        double h2 = 0.0, e2 = 0.0;
        bool ovf = false;
        uint2* out = reinterpret_cast<uint2*>(a.Xh + row * a.Kp);
#pragma unroll
        for (int j = 0; j < GPL; ++j) {
            const int g = 4 * j + l4;
            if (g < ng) {
                const float xc[4] = {x[j].x, x[j].y, x[j].z, x[j].w};
                __half hq[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    __half h = __float2half_rn(0.f);
                    if (real) {
                        const float t = __fsub_rn(xc[e], a.mu[4 * g + e]) * s;
                        h = __float2half_rn(t);
                        const double hv = static_cast<double>(__half2float(h));
                        const double err = fabs(hv - static_cast<double>(t)) + fabs(static_cast<double>(t)) * 0x1.0p-23;
                        h2 += hv * hv;
                        e2 += err * err;
                        if (QUERY) {
                            h = __float2half_rn(-2.f * __half2float(h));
                            ovf |= __hisinf(h) != 0;
                        }
                    }
                    hq[e] = h;
                }
                if (inpad) {
                    uint2 w;
                    w.x = static_cast<uint32_t>(__half_as_ushort(hq[0])) | (static_cast<uint32_t>(__half_as_ushort(hq[1])) << 16);
                    w.y = static_cast<uint32_t>(__half_as_ushort(hq[2])) | (static_cast<uint32_t>(__half_as_ushort(hq[3])) << 16);
                    out[g] = w;
                }
            }
        }
#pragma unroll
        for (int o = 1; o < 4; o <<= 1) {
            h2 += __shfl_xor_sync(0xffffffffu, h2, o);
            e2 += __shfl_xor_sync(0xffffffffu, e2, o);
        }
        const bool any_ovf = (__ballot_sync(0xffffffffu, ovf) >> (lane & ~3) & 0xfu) != 0;
        const float delta = any_ovf ? kInf : static_cast<float>(sqrt(e2) * (1.0 + 0x1.0p-20)) * (1.f + 1e-6f);
        const float xn = static_cast<float>(sqrt(h2)) * (1.f + 1e-6f);
        // tail columns [d, Kp): zeros, or the three folded-norm columns
        __half nc[3];
        if (QUERY) {
            nc[0] = nc[1] = nc[2] = __float2half_rn(1.f);
        } else if (real) {
            nc[0] = __double2half(h2);
            const double r1 = h2 - static_cast<double>(__half2float(nc[0]));
            nc[1] = __double2half(r1);
            nc[2] = __double2half(r1 - static_cast<double>(__half2float(nc[1])));
        } else {
            nc[0] = __float2half_rn(kInf);  // padding: A = +inf
            nc[1] = nc[2] = __float2half_rn(0.f);
        }
        if (inpad)
            for (int g = ng + l4; g < nk; g += 4) {
                unsigned short hv[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int c = 4 * g + e;
                    const int nci = c - a.norm_col;
                    hv[e] = (a.norm_col >= 0 && nci >= 0 && nci < 3) ? __half_as_ushort(nc[nci]) : 0;
                }
                out[g] = make_uint2(hv[0] | (static_cast<uint32_t>(hv[1]) << 16),
                                    hv[2] | (static_cast<uint32_t>(hv[3]) << 16));
            }
        if (inpad && l4 == 0) {
            if (QUERY) {
                a.qconst[row] = make_float4(static_cast<float>(h2), delta, xn, 0.f);
                if (a.tinit) a.tinit[row] = 0xffffffffu;
            } else if (a.norm_col < 0) {
                a.norm[row] = real ? static_cast<float>(h2) : kInf;
            }
        }
        if (!QUERY && real) {
            dmax = fmaxf(dmax, delta);
            nmax = fmaxf(nmax, xn);
        }
    }
    if (!QUERY) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            dmax = fmaxf(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
            nmax = fmaxf(nmax, __shfl_xor_sync(0xffffffffu, nmax, o));
        }
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
            atomicMax(a.gmax + 0, __float_as_uint(dm));
            atomicMax(a.gmax + 1, __float_as_uint(nm));
        }
    }
}

}  // namespace

void launch_range(const float* X, int64_t rows, int d, unsigned* mn, unsigned* mx,
                  cudaStream_t stream) {
    ProfileScope ps(stream, "prep_range_kernel");
    const int vec = (d % 4 == 0) ? 4 : 1;
    const int rpb = 256 / (d / vec);
    const int64_t want = (rows + rpb * 8 - 1) / (rpb * 8);  // >= 8 rows per thread
    const unsigned grid =
        static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(want, 4 * kSmCount)));
    if (vec == 4)
        range_kernel<4><<<grid, 256, 0, stream>>>(X, rows, d, mn, mx);
    else
        range_kernel<1><<<grid, 256, 0, stream>>>(X, rows, d, mn, mx);
    KNN_LAUNCH_CHECK();
}

void launch_scale(const unsigned* mn, const unsigned* mx, int d, int Kp, float* mu, float* scale,
                  unsigned* gmax, cudaStream_t stream) {
    {
        ProfileScope ps(stream, "prep_scale_kernel");
        scale_kernel<<<1, 256, 0, stream>>>(mn, mx, d, Kp, mu, scale, gmax);
    }
    KNN_LAUNCH_CHECK();
}

void launch_convert(const PrepArgs& pr, bool query, cudaStream_t stream) {
    if (pr.d % 4 == 0 && pr.d <= 128 && std::getenv("KNN_B200_CONVERT_V1") == nullptr) {
        // 64 rows per block step; enough blocks to fill the SMs several times over
        const unsigned grid =
            static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>((pr.rows_pad + 63) / 64, 16 * kSmCount)));
        const int gpl = (pr.d / 4 + 3) / 4;
        ProfileScope ps(stream, query ? "prep_convert_queries" : "prep_convert_refs");
        auto go = [&](auto kq, auto kr) {
            (void)kq;
            (void)kr;
            convert4_kernel<decltype(kq)::value, decltype(kr)::value><<<grid, 256, 0, stream>>>(pr);
        };
        using T = std::true_type;
        using F = std::false_type;
        if (gpl <= 2) query ? go(T{}, std::integral_constant<int, 2>{}) : go(F{}, std::integral_constant<int, 2>{});
        else if (gpl <= 4) query ? go(T{}, std::integral_constant<int, 4>{}) : go(F{}, std::integral_constant<int, 4>{});
        else if (gpl <= 6) query ? go(T{}, std::integral_constant<int, 6>{}) : go(F{}, std::integral_constant<int, 6>{});
        else query ? go(T{}, std::integral_constant<int, 8>{}) : go(F{}, std::integral_constant<int, 8>{});
        KNN_LAUNCH_CHECK();
        return;
    }
    const unsigned grid =
        static_cast<unsigned>(std::min<int64_t>((pr.rows_pad + 7) / 8, 8 * kSmCount));
    {
        ProfileScope ps(stream, query ? "prep_convert_queries" : "prep_convert_refs");
        if (query)
            convert_kernel<true><<<grid, 256, 0, stream>>>(pr);
        else
            convert_kernel<false><<<grid, 256, 0, stream>>>(pr);
    }
    KNN_LAUNCH_CHECK();
}

}  // namespace tp
}  // namespace knnb200
