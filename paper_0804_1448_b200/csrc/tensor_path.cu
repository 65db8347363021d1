// tensor_path.cu -- placeholder until the tcgen05 candidate kernel lands.
#include "common.cuh"
#include "engine.cuh"
#include "tensor_path.cuh"

namespace knnb200 {

bool tensor_path_supported(int64_t, int64_t, int, int) { return false; }

void run_tensor_path(DeviceContext&, cudaStream_t, const float*, int64_t, const float*, int64_t,
                     int, int, int, int64_t, float*, int64_t*) {
    throw CudaError("tensor path not built");
}

}  // namespace knnb200
