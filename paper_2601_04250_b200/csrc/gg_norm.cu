// gg_norm.cu — LayerNorm and DistilBERT embedding+LayerNorm (HBM-bound, one warp per row).
#include "gg_common.cuh"
#include "gg_kernels.h"
#include <cuda_bf16.h>

namespace gg {

template <int PER_LANE>  // elements per lane (width / 32), multiple of 8
__device__ __forceinline__ void ln_row(float (&x)[PER_LANE], int width, const float* gamma,
                                       const float* beta, float eps, __nv_bfloat16* y) {
  const int lane = threadIdx.x & 31;
  float sum = 0.f;
#pragma unroll
  for (int i = 0; i < PER_LANE; ++i) sum += x[i];
#pragma unroll
  for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  const float mean = sum / width;
  float var = 0.f;
#pragma unroll
  for (int i = 0; i < PER_LANE; ++i) {
    const float d = x[i] - mean;
    var += d * d;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) var += __shfl_xor_sync(0xffffffffu, var, o);
  const float rstd = rsqrtf(var / width + eps);
#pragma unroll
  for (int c = 0; c < PER_LANE / 8; ++c) {
    const int col = (c * 32 + lane) * 8;
    const float4 g0 = __ldg(reinterpret_cast<const float4*>(gamma + col));
    const float4 g1 = __ldg(reinterpret_cast<const float4*>(gamma + col + 4));
    const float4 b0 = __ldg(reinterpret_cast<const float4*>(beta + col));
    const float4 b1 = __ldg(reinterpret_cast<const float4*>(beta + col + 4));
    const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
    const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
    float o[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) o[e] = (x[c * 8 + e] - mean) * rstd * gg[e] + bb[e];
    uint4 u;
    __nv_bfloat162 t0 = __floats2bfloat162_rn(o[0], o[1]), t1 = __floats2bfloat162_rn(o[2], o[3]);
    __nv_bfloat162 t2 = __floats2bfloat162_rn(o[4], o[5]), t3 = __floats2bfloat162_rn(o[6], o[7]);
    u.x = *reinterpret_cast<uint32_t*>(&t0);
    u.y = *reinterpret_cast<uint32_t*>(&t1);
    u.z = *reinterpret_cast<uint32_t*>(&t2);
    u.w = *reinterpret_cast<uint32_t*>(&t3);
    *reinterpret_cast<uint4*>(y + col) = u;
  }
}

template <int PER_LANE>
__device__ __forceinline__ void load_row(const __nv_bfloat16* src, float (&x)[PER_LANE], bool add) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int c = 0; c < PER_LANE / 8; ++c) {
    const uint4 u = __ldg(reinterpret_cast<const uint4*>(src + (c * 32 + lane) * 8));
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = __bfloat1622float2(h[e]);
      if (add) {
        x[c * 8 + 2 * e] += f.x;
        x[c * 8 + 2 * e + 1] += f.y;
      } else {
        x[c * 8 + 2 * e] = f.x;
        x[c * 8 + 2 * e + 1] = f.y;
      }
    }
  }
}

// A warp normalizes kLnRowsPerWarp rows in turn with its lanes' gamma / beta held
// in registers (loaded once, not once per row: per-row reloads made this kernel
// L1-throughput-bound, ncu l1tex 73 %), the next row's load issued before the
// current row's reductions.  Launched with programmatic dependent launch.
constexpr int kLnRowsPerWarp = 4;
constexpr int kLnWarps = 4;
template <int PER_LANE>
__global__ void __launch_bounds__(32 * kLnWarps) layernorm_kernel(const __nv_bfloat16* x, int64_t ldx,
                                                                 __nv_bfloat16* y, int64_t ldy,
                                                                 const float* gamma, const float* beta,
                                                                 int64_t rows, int width, float eps,
                                                                 const int32_t* count, int rows_per_item) {
  const int lane = threadIdx.x & 31;
  float g[PER_LANE], bt[PER_LANE];
#pragma unroll
  for (int c = 0; c < PER_LANE / 8; ++c) {
    const int col = (c * 32 + lane) * 8;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const float4 gg4 = __ldg(reinterpret_cast<const float4*>(gamma + col) + h);
      const float4 bb4 = __ldg(reinterpret_cast<const float4*>(beta + col) + h);
      g[c * 8 + 4 * h + 0] = gg4.x; g[c * 8 + 4 * h + 1] = gg4.y;
      g[c * 8 + 4 * h + 2] = gg4.z; g[c * 8 + 4 * h + 3] = gg4.w;
      bt[c * 8 + 4 * h + 0] = bb4.x; bt[c * 8 + 4 * h + 1] = bb4.y;
      bt[c * 8 + 4 * h + 2] = bb4.z; bt[c * 8 + 4 * h + 3] = bb4.w;
    }
  }
  griddep_wait();
  griddep_launch();
  if (count) rows = min(rows, (int64_t)__ldg(count) * rows_per_item);
  const int64_t r0 = ((int64_t)blockIdx.x * kLnWarps + (threadIdx.x >> 5)) * kLnRowsPerWarp;
  if (r0 >= rows) return;
  float v[PER_LANE], nx[PER_LANE];
  load_row<PER_LANE>(x + r0 * ldx, v, false);
#pragma unroll 1
  for (int j = 0; j < kLnRowsPerWarp; ++j) {
    const int64_t r = r0 + j;
    if (r >= rows) break;
    if (j + 1 < kLnRowsPerWarp && r + 1 < rows) load_row<PER_LANE>(x + (r + 1) * ldx, nx, false);
    float sum = 0.f;
#pragma unroll
    for (int i = 0; i < PER_LANE; ++i) sum += v[i];
#pragma unroll
    for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    const float mean = sum / width;
    float var = 0.f;
#pragma unroll
    for (int i = 0; i < PER_LANE; ++i) {
      const float d = v[i] - mean;
      var += d * d;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) var += __shfl_xor_sync(0xffffffffu, var, o);
    const float rstd = rsqrtf(var / width + eps);
    __nv_bfloat16* yr = y + r * ldy;
#pragma unroll
    for (int c = 0; c < PER_LANE / 8; ++c) {
      const int col = (c * 32 + lane) * 8;
      float o8[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) o8[e] = (v[c * 8 + e] - mean) * rstd * g[c * 8 + e] + bt[c * 8 + e];
      uint4 u;
      __nv_bfloat162 t0 = __floats2bfloat162_rn(o8[0], o8[1]), t1 = __floats2bfloat162_rn(o8[2], o8[3]);
      __nv_bfloat162 t2 = __floats2bfloat162_rn(o8[4], o8[5]), t3 = __floats2bfloat162_rn(o8[6], o8[7]);
      u.x = *reinterpret_cast<uint32_t*>(&t0);
      u.y = *reinterpret_cast<uint32_t*>(&t1);
      u.z = *reinterpret_cast<uint32_t*>(&t2);
      u.w = *reinterpret_cast<uint32_t*>(&t3);
      *reinterpret_cast<uint4*>(yr + col) = u;
    }
#pragma unroll
    for (int i = 0; i < PER_LANE; ++i) v[i] = nx[i];
  }
}

template <int PER_LANE>
__global__ void __launch_bounds__(256) embed_ln_kernel(const int32_t* ids, const __nv_bfloat16* word,
                                                       const __nv_bfloat16* pos, __nv_bfloat16* y,
                                                       const float* gamma, const float* beta,
                                                       int64_t tokens, int seq_len, int width,
                                                       float eps, const int32_t* count) {
  griddep_wait();
  griddep_launch();
  const int64_t t = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (count) tokens = min(tokens, (int64_t)__ldg(count) * seq_len);
  if (t >= tokens) return;
  float v[PER_LANE];
  load_row<PER_LANE>(word + (int64_t)__ldg(ids + t) * width, v, false);
  load_row<PER_LANE>(pos + (int64_t)(t % seq_len) * width, v, true);
  ln_row<PER_LANE>(v, width, gamma, beta, eps, y + t * width);
}

}  // namespace gg

using namespace gg;

extern "C" int gg_layernorm(const void* x, int64_t ldx, void* y, int64_t ldy, const float* gamma,
                            const float* beta, int64_t rows, int32_t width, float eps,
                            const int32_t* count_dev, int32_t rows_per_item, void* stream) {
  if (!x || !y || !gamma || !beta || rows < 0) return GG_ERR_INVALID_ARGUMENT;
  if (width != 768 || ldx % 8 || ldy % 8) return GG_ERR_UNSUPPORTED;
  if (rows == 0) return GG_OK;
  const int64_t per_block = kLnWarps * kLnRowsPerWarp;
  if (launch_pdl(layernorm_kernel<24>, dim3((unsigned)((rows + per_block - 1) / per_block)), dim3(32 * kLnWarps), 0,
                 gg_stream(stream), reinterpret_cast<const __nv_bfloat16*>(x), ldx,
                 reinterpret_cast<__nv_bfloat16*>(y), ldy, gamma, beta, rows, width, eps, count_dev,
                 rows_per_item) != cudaSuccess)
    return GG_ERR_CUDA;
  GG_LAUNCH_OK();
  return GG_OK;
}

extern "C" int gg_embed_layernorm(const int32_t* ids, const void* word, const void* pos, void* y,
                                  const float* gamma, const float* beta, int64_t tokens,
                                  int32_t seq_len, int32_t width, float eps,
                                  const int32_t* count_dev, void* stream) {
  if (!ids || !word || !pos || !y || !gamma || !beta || tokens < 0 || seq_len <= 0)
    return GG_ERR_INVALID_ARGUMENT;
  if (width != 768) return GG_ERR_UNSUPPORTED;
  if (tokens == 0) return GG_OK;
  if (launch_pdl(embed_ln_kernel<24>, dim3((unsigned)((tokens + 7) / 8)), dim3(256), 0, gg_stream(stream),
                 ids, reinterpret_cast<const __nv_bfloat16*>(word), reinterpret_cast<const __nv_bfloat16*>(pos),
                 reinterpret_cast<__nv_bfloat16*>(y), gamma, beta, tokens, seq_len, width, eps,
                 count_dev) != cudaSuccess)
    return GG_ERR_CUDA;
  GG_LAUNCH_OK();
  return GG_OK;
}
