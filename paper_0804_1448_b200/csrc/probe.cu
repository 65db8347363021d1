// probe.cu -- minimal tcgen05 GEMM used by the GPU tests to validate the
// building blocks the tensor path relies on (TMA SWIZZLE_128B loads, smem
// matrix descriptors with K-slice advance, instruction descriptor, TMEM
// allocation and the 32x32b load layout): D[128x128] = A[128xK] * B[128xK]^T.
#include "../../include/knn_b200.h"
#include "common.cuh"
#include "profile.cuh"
#include "sm100.cuh"
#include "tmap.cuh"

namespace knnb200 {

namespace {

__global__ void __launch_bounds__(128) mma_probe_kernel(const __grid_constant__ CUtensorMap ta,
                                                        const __grid_constant__ CUtensorMap tb,
                                                        int K, float* D) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1024-align the operand tiles (SWIZZLE_128B atoms)
    unsigned char* base = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    const int KB = (K + 63) / 64;
    unsigned char* As = base;
    unsigned char* Bs = base + KB * 16384;
    __shared__ uint64_t bar_load, bar_mma;
    __shared__ uint32_t tmem_base;

    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        sm100::mbar_init(&bar_load, 1);
        sm100::mbar_init(&bar_mma, 1);
        sm100::fence_mbar_init();
    }
    if (warp == 1) sm100::tmem_alloc(&tmem_base, 128);
    sm100::tc_fence_before();
    __syncthreads();
    sm100::tc_fence_after();
    const uint32_t tmem = tmem_base;

    if (threadIdx.x == 0) {
        sm100::mbar_expect_tx(&bar_load, 2u * KB * 16384u);
        for (int kb = 0; kb < KB; ++kb) {
            sm100::tma_load_2d(As + kb * 16384, &ta, &bar_load, kb * 64, 0);
            sm100::tma_load_2d(Bs + kb * 16384, &tb, &bar_load, kb * 64, 0);
        }
        sm100::mbar_wait(&bar_load, 0);
        sm100::tc_fence_after();
        const uint32_t idesc = sm100::idesc_f16_f32(128, 128);
        for (int ks = 0; ks < K / 16; ++ks) {
            const int kb = ks >> 2, w = ks & 3;
            const uint64_t ad = sm100::sdesc_k_sw128(sm100::smem_u32(As + kb * 16384 + w * 32));
            const uint64_t bd = sm100::sdesc_k_sw128(sm100::smem_u32(Bs + kb * 16384 + w * 32));
            sm100::mma_f16_ss(tmem, ad, bd, idesc, ks > 0 ? 1u : 0u);
        }
        sm100::mma_commit(&bar_mma);
    }
    __syncwarp();
    sm100::mbar_wait(&bar_mma, 0);
    sm100::tc_fence_after();
    const int row = warp * 32 + (threadIdx.x & 31);
    for (int c = 0; c < 4; ++c) {
        uint32_t r[32];
        sm100::tmem_ld_32x32b_x32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c * 32, r);
        sm100::tmem_ld_wait();
        for (int j = 0; j < 32; ++j) D[row * 128 + c * 32 + j] = __uint_as_float(r[j]);
    }
    sm100::tc_fence_before();
    __syncthreads();
    if (warp == 1) sm100::tmem_dealloc(tmem, 128);
}

}  // namespace
}  // namespace knnb200

using namespace knnb200;

extern "C" KNN_B200_API knn_b200_status knn_b200_debug_mma_probe(const void* dA, const void* dB,
                                                                 int32_t K, float* dD) {
    try {
        if (K <= 0 || K % 16 || K > 256) return KNN_B200_EINVAL;
        const CUtensorMap ta = make_tmap_f16_sw128(dA, 128, K, 128, 64);
        const CUtensorMap tb = make_tmap_f16_sw128(dB, 128, K, 128, 64);
        const int KB = (K + 63) / 64;
        const size_t smem = 2 * KB * 16384 + 1024;
        KNN_CUDA_CHECK(cudaFuncSetAttribute(mma_probe_kernel,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            static_cast<int>(smem)));
        mma_probe_kernel<<<1, 128, smem>>>(ta, tb, K, dD);
        KNN_LAUNCH_CHECK();
        KNN_CUDA_CHECK(cudaDeviceSynchronize());
        return KNN_B200_OK;
    } catch (const std::exception& e) {
        return KNN_B200_ECUDA;
    }
}
