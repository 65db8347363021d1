// tmap.cuh -- TMA tensor-map construction (host).
#pragma once

#include <cuda.h>
#include <stdint.h>

namespace knnb200 {

CUtensorMap make_tmap_f16_sw128(const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows,
                                uint32_t box_cols);
// the 16-column K tail: columns [col0, col0 + 16) of a row-major fp16 matrix
// with row pitch `pitch` elements, box {16, box_rows}, SWIZZLE_32B
CUtensorMap make_tmap_f16_tail16(const void* base, uint64_t rows, uint64_t pitch, uint64_t col0,
                                 uint32_t box_rows);

}  // namespace knnb200
