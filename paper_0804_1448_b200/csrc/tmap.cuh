// tmap.cuh -- TMA tensor-map construction (host).
#pragma once

#include <cuda.h>
#include <stdint.h>

namespace knnb200 {

CUtensorMap make_tmap_f16_sw128(const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows,
                                uint32_t box_cols);

}  // namespace knnb200
