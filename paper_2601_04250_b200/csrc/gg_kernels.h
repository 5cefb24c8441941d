// gg_kernels.h — internal host helpers shared by the forward-pass translation units.
#pragma once
#include <cuda.h>
#include <stdint.h>

namespace gg {
// 2-D bf16 K-major TMA map: [rows, cols], row pitch ld elements, box [64, box_rows], SW128.
int make_map_2d(CUtensorMap* map, const void* ptr, int64_t rows, int64_t cols, int64_t ld,
                int box_rows);
int num_sms();
}  // namespace gg
