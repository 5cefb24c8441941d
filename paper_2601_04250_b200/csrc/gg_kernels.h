// gg_kernels.h — internal host helpers shared by the forward-pass translation units.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <utility>

namespace gg {
// 2-D bf16 K-major TMA map: [rows, cols], row pitch ld elements, box [64, box_rows], SW128.
int make_map_2d(CUtensorMap* map, const void* ptr, int64_t rows, int64_t cols, int64_t ld,
                int box_rows);
int num_sms();

// Programmatic dependent launch: the kernel may start (prologue: barriers, TMEM,
// weight loads) while its stream predecessor drains; it must execute
// griddep_wait() before touching anything the predecessor produces or reads.
// GG_NO_PDL=1 falls back to ordinary stream serialization.
inline bool pdl_enabled() {
  static int on = -1;
  if (on < 0) on = getenv("GG_NO_PDL") ? 0 : 1;
  return on == 1;
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t stream, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
}  // namespace gg

// kern<<<grid, block, smem, stream>>>(args...) with the PDL attribute; returns
// GG_ERR_CUDA from the enclosing function on a launch error.
#define GG_PDL_LAUNCH(kern, grid, block, smem, stream, ...)                                  \
  do {                                                                                       \
    if (::gg::launch_pdl(kern, dim3(grid), dim3(block), (size_t)(smem), (stream), __VA_ARGS__) != \
        cudaSuccess)                                                                         \
      return GG_ERR_CUDA;                                                                    \
  } while (0)
