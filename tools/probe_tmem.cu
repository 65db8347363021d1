// Dev microbenchmark (GPU): tcgen05.ld throughput per SM as a function of the
// number of loading warps and the load width.  Not part of the product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I. tools/probe_tmem.cu -o /tmp/probe_tmem -lcuda
#include <cstdio>

#include "../paper_0804_1448_b200/csrc/sm100.cuh"

using namespace knnb200;

template <int X>
__device__ __forceinline__ void ld_chunk(uint32_t taddr, float& acc);

template <>
__device__ __forceinline__ void ld_chunk<32>(uint32_t taddr, float& acc) {
    uint32_t r[32];
    sm100::tmem_ld_32x32b_x32(taddr, r);
    sm100::tmem_ld_wait();
#pragma unroll
    for (int j = 0; j < 32; ++j) acc += __uint_as_float(r[j]);
}

// two x32 loads in flight before one wait
template <>
__device__ __forceinline__ void ld_chunk<64>(uint32_t taddr, float& acc) {
    uint32_t r[32], s[32];
    sm100::tmem_ld_32x32b_x32(taddr, r);
    sm100::tmem_ld_32x32b_x32(taddr + 32, s);
    sm100::tmem_ld_wait();
#pragma unroll
    for (int j = 0; j < 32; ++j) acc += __uint_as_float(r[j]) + __uint_as_float(s[j]);
}

template <int X>
__global__ void probe(int iters, unsigned long long* cyc, float* sink) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) sm100::tmem_alloc(&slot, 512);
    sm100::tc_fence_before();
    __syncthreads();
    sm100::tc_fence_after();
    const uint32_t tmem = slot;
    const uint32_t base = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16);
    float acc = 0.f;
    __syncthreads();
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        const uint32_t col = static_cast<uint32_t>((i * X + (warp >> 2) * 64) & 511);
        ld_chunk<X>(base + col, acc);
    }
    __syncthreads();
    const long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = static_cast<unsigned long long>(t1 - t0);
    if (acc == 1.2345f) sink[0] = acc;
    sm100::tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        sm100::tc_fence_after();
        sm100::tmem_dealloc(tmem, 512);
    }
}

int main() {
    unsigned long long* cyc;
    float* sink;
    cudaMalloc(&cyc, sizeof(unsigned long long) * 148);
    cudaMalloc(&sink, 4);
    const int iters = 4096;
    for (int x : {32, 64}) {
        for (int warps : {4, 8, 12, 16}) {
            auto k = x == 32 ? probe<32> : probe<64>;
            k<<<148, warps * 32>>>(iters, cyc, sink);
            k<<<148, warps * 32>>>(iters, cyc, sink);
            cudaError_t e = cudaDeviceSynchronize();
            unsigned long long h[148];
            cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
            double bytes = static_cast<double>(iters) * warps * 32 * x * 4;
            printf("x=%d warps=%2d: %8llu cycles, %.1f B/cycle/SM (%s)\n", x, warps, h[0],
                   bytes / h[0], cudaGetErrorString(e));
        }
    }
    return 0;
}
