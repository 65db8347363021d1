// tmap.cu -- host-side TMA tensor-map encoding through the driver entry point
// (no link-time dependency on libcuda; resolved via cudaGetDriverEntryPoint).
#include <cudaTypedefs.h>

#include <mutex>

#include "common.cuh"
#include "tmap.cuh"

namespace knnb200 {

namespace {
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    if (!fn) throw CudaError("cuTensorMapEncodeTiled unavailable");
    return fn;
}
}  // namespace

// Row-major fp16 matrix [rows][cols] (cols contiguous, row pitch = cols*2 B,
// a multiple of 16).  Box = {box_cols, box_rows} with SWIZZLE_128B
// (box_cols * 2 must be 128).  Out-of-bounds elements read as zero.
CUtensorMap make_tmap_f16_sw128(const void* base, uint64_t rows, uint64_t cols,
                                uint32_t box_rows, uint32_t box_cols) {
    CUtensorMap m;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {cols * 2};
    cuuint32_t box[2] = {box_cols, box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base), dims,
                             strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        throw CudaError("cuTensorMapEncodeTiled failed with CUresult " + std::to_string(r));
    return m;
}

CUtensorMap make_tmap_f16_tail16(const void* base, uint64_t rows, uint64_t pitch, uint64_t col0,
                                 uint32_t box_rows) {
    CUtensorMap m;
    cuuint64_t dims[2] = {16, rows};
    cuuint64_t strides[1] = {pitch * 2};
    cuuint32_t box[2] = {16, box_rows};
    cuuint32_t estr[2] = {1, 1};
    void* p = const_cast<char*>(static_cast<const char*>(base) + col0 * 2);
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, p, dims, strides, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        throw CudaError("cuTensorMapEncodeTiled (tail) failed with CUresult " + std::to_string(r));
    return m;
}

}  // namespace knnb200
