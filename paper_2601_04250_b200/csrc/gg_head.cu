// gg_head.cu — DistilBERT classification head as ONE launch: LayerNorm of the B CLS rows
// (optional), pre_classifier (768 x 768) + bias + ReLU, classifier (768 -> labels) + bias.
//
// HF DistilBertForSequenceClassification.forward: hidden[:, 0] -> pre_classifier -> ReLU
// -> dropout (identity in eval) -> classifier.  The head is latency-bound (B = 128 rows,
// 0.2 GFLOP): as three launches (LayerNorm, two single-CTA-tile GEMMs) it cost ~20 us of
// a serving step, mostly launch and pipeline fill.  Here a 2-D grid of CTAs (16 CLS rows x
// 96 pre_classifier columns each, 64 CTAs at B = 128) stages its weight slice with cp.async
// BEFORE the programmatic-dependent-launch wait (the weights do not depend on the encoder),
// normalises its 16 rows into shared memory exactly as gg_layernorm does (same bf16
// operand), runs the 16 x 96 x 768 product on mma.sync (bf16, fp32 accumulate; the tile is
// far too small for tcgen05 to pay), applies bias + ReLU + the bf16 rounding of the pooled
// activation, and reduces its classifier partial dot products; the 8 column-block CTAs of a
// row block form a thread-block cluster and CTA 0 adds their partials from its shared
// memory (written over DSMEM) in a fixed order — the logits are deterministic.
#include "gg_common.cuh"
#include "gg_kernels.h"
#include "gg_tc.cuh"
#include <cuda_bf16.h>

namespace gg {
using tc::smem_u32;

constexpr int kHeadD = 768;
constexpr int kHeadRows = 16;              // CLS rows per CTA (one m16 MMA tile)
constexpr int kHeadCols = 96;              // pre_classifier columns per CTA (12 n8 tiles)
constexpr int kHeadColBlocks = kHeadD / kHeadCols;
constexpr int kHeadLd = kHeadD + 8;        // padded smem row (bf16): ldmatrix conflict-free
constexpr int kHeadThreads = 256;
constexpr int kHeadMaxLabels = 32;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}

__device__ __forceinline__ void ldsm_x4(const void* p, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(smem_u32(p)));
}

__device__ __forceinline__ void mma_bf16_16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
               "{%0,%1,%2,%3};"
               : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// Shared memory: W_pre slice [96][kHeadLd] bf16 | CLS operand [16][kHeadLd] bf16 |
// gamma, beta [768] fp32 | W_cls slice [labels][96] fp32 | classifier partials of
// the cluster's 8 CTAs [8][16][kHeadMaxLabels] fp32 (written into CTA 0's copy).
constexpr size_t kHeadOffA = (size_t)kHeadCols * kHeadLd * 2;
constexpr size_t kHeadOffG = kHeadOffA + (size_t)kHeadRows * kHeadLd * 2;
constexpr size_t kHeadOffWc = kHeadOffG + 2 * kHeadD * 4;
constexpr size_t kHeadOffP = kHeadOffWc + (size_t)kHeadMaxLabels * kHeadCols * 4;
constexpr size_t kHeadSmemAll = kHeadOffP + (size_t)kHeadColBlocks * kHeadRows * kHeadMaxLabels * 4;

// One cluster per 16-row block: its 8 CTAs are the 96-column blocks of the
// pre_classifier; their classifier partials meet in CTA 0's shared memory over
// DSMEM (fixed summation order, no global round trip).
__global__ void __cluster_dims__(kHeadColBlocks, 1, 1) __launch_bounds__(kHeadThreads, 1)
cls_head_kernel(const __nv_bfloat16* __restrict__ hidden, int64_t ld_rows, const float* __restrict__ ln_g,
                const float* __restrict__ ln_b, float eps, const __nv_bfloat16* __restrict__ w_pre,
                const float* __restrict__ b_pre, const __nv_bfloat16* __restrict__ w_cls,
                const float* __restrict__ b_cls, int labels, float* __restrict__ logits, int64_t ld_logits,
                int rows, const int32_t* __restrict__ count) {
  extern __shared__ __align__(128) uint8_t head_smem[];
  __nv_bfloat16* sw = reinterpret_cast<__nv_bfloat16*>(head_smem);
  __nv_bfloat16* sa = reinterpret_cast<__nv_bfloat16*>(head_smem + kHeadOffA);
  float* sg = reinterpret_cast<float*>(head_smem + kHeadOffG);       // gamma | beta
  float* swc = reinterpret_cast<float*>(head_smem + kHeadOffWc);     // [labels][96]
  float* spart = reinterpret_cast<float*>(head_smem + kHeadOffP);    // [8][16][kHeadMaxLabels]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int cb = blockIdx.x, rb = blockIdx.y;
  const int n0 = cb * kHeadCols;
  // everything that does not depend on the encoder, before the dependency wait:
  // the W_pre slice (cp.async), gamma / beta, the W_cls slice
  for (int i = tid; i < kHeadCols * (kHeadD / 8); i += kHeadThreads) {
    const int r = i / (kHeadD / 8), c = (i % (kHeadD / 8)) * 8;
    cp_async16(sw + r * kHeadLd + c, w_pre + (int64_t)(n0 + r) * kHeadD + c);
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  if (ln_g)
    for (int i = tid; i < kHeadD; i += kHeadThreads) {
      sg[i] = __ldg(ln_g + i);
      sg[kHeadD + i] = __ldg(ln_b + i);
    }
  for (int i = tid; i < labels * kHeadCols; i += kHeadThreads)
    swc[i] = __bfloat162float(__ldg(w_cls + (int64_t)(i / kHeadCols) * kHeadD + n0 + i % kHeadCols));
  griddep_wait();
  griddep_launch();
  if (count) rows = min(rows, (int)__ldg(count));
  const int r0 = rb * kHeadRows;
  if (r0 >= rows) {   // the whole cluster (one row block) leaves together
    asm volatile("cp.async.wait_all;" ::: "memory");
    return;
  }
  __syncthreads();   // gamma / beta visible
  // the CTA's CLS rows -> bf16 operand (LayerNorm as gg_layernorm computes it);
  // warp w takes rows w and w + 8, both rows' loads in flight before the reductions
  {
    float v[2][24];
    bool have[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = r0 + warp + 8 * h;
      have[h] = r < rows;
      const __nv_bfloat16* src = hidden + (int64_t)(have[h] ? r : r0) * ld_rows;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const uint4 u = __ldcg(reinterpret_cast<const uint4*>(src + (c * 32 + lane) * 8));
        const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __bfloat1622float2(h2[e]);
          v[h][c * 8 + 2 * e] = f.x;
          v[h][c * 8 + 2 * e + 1] = f.y;
        }
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      __nv_bfloat16* dst = sa + (warp + 8 * h) * kHeadLd;
      if (!have[h]) {
        for (int c = lane * 8; c < kHeadD; c += 256) *reinterpret_cast<uint4*>(dst + c) = make_uint4(0, 0, 0, 0);
        continue;
      }
      float mean = 0.f, rstd = 1.f;
      if (ln_g) {
        float sum = 0.f;
#pragma unroll
        for (int i = 0; i < 24; ++i) sum += v[h][i];
#pragma unroll
        for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        mean = sum / kHeadD;
        float var = 0.f;
#pragma unroll
        for (int i = 0; i < 24; ++i) {
          const float d = v[h][i] - mean;
          var += d * d;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) var += __shfl_xor_sync(0xffffffffu, var, o);
        rstd = rsqrtf(var / kHeadD + eps);
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const int col = (c * 32 + lane) * 8;
        uint32_t w[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float x0 = v[h][c * 8 + 2 * e], x1 = v[h][c * 8 + 2 * e + 1];
          if (ln_g) {
            x0 = (x0 - mean) * rstd * sg[col + 2 * e] + sg[kHeadD + col + 2 * e];
            x1 = (x1 - mean) * rstd * sg[col + 2 * e + 1] + sg[kHeadD + col + 2 * e + 1];
          }
          __nv_bfloat162 t = __floats2bfloat162_rn(x0, x1);
          w[e] = *reinterpret_cast<uint32_t*>(&t);
        }
        *reinterpret_cast<uint4*>(dst + col) = make_uint4(w[0], w[1], w[2], w[3]);
      }
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  // 16 x 96 x 768 on mma.sync: warp w owns k in [96 w, 96 w + 96), all 12 n8 tiles
  float acc[12][4];
#pragma unroll
  for (int t = 0; t < 12; ++t) acc[t][0] = acc[t][1] = acc[t][2] = acc[t][3] = 0.f;
  const int kw = warp * (kHeadD / 8);
#pragma unroll
  for (int ks = 0; ks < kHeadD / 8 / 16; ++ks) {
    const int k = kw + ks * 16;
    uint32_t a[4];
    ldsm_x4(sa + (lane & 15) * kHeadLd + k + (lane >> 4) * 8, a[0], a[1], a[2], a[3]);
#pragma unroll
    for (int t = 0; t < 12; t += 2) {
      uint32_t b0, b1, b2, b3;
      ldsm_x4(sw + (t * 8 + (lane & 7) + (lane >> 4) * 8) * kHeadLd + k + ((lane >> 3) & 1) * 8, b0, b1, b2, b3);
      mma_bf16_16816(acc[t], a, b0, b1);
      mma_bf16_16816(acc[t + 1], a, b2, b3);
    }
  }
  __syncthreads();  // weights no longer needed: reuse as the split-K reduction buffer
  float* red = reinterpret_cast<float*>(head_smem);                 // [8 warps][16][96]
  {
    const int g = lane >> 2, q = (lane & 3) * 2;
    float* rw = red + warp * kHeadRows * kHeadCols;
#pragma unroll
    for (int t = 0; t < 12; ++t) {
      rw[g * kHeadCols + t * 8 + q] = acc[t][0];
      rw[g * kHeadCols + t * 8 + q + 1] = acc[t][1];
      rw[(g + 8) * kHeadCols + t * 8 + q] = acc[t][2];
      rw[(g + 8) * kHeadCols + t * 8 + q + 1] = acc[t][3];
    }
  }
  __syncthreads();
  float* pooled = red + 8 * kHeadRows * kHeadCols;                  // [16][96] fp32 of bf16
  for (int i = tid; i < kHeadRows * kHeadCols; i += kHeadThreads) {
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) s += red[w * kHeadRows * kHeadCols + i];
    s = fmaxf(s + __ldg(b_pre + n0 + i % kHeadCols), 0.f);
    pooled[i] = __bfloat162float(__float2bfloat16_rn(s));
  }
  __syncthreads();
  // classifier partials over this CTA's 96 columns -> CTA 0's spart[cb] (DSMEM)
  const uint32_t part0 = tc::mapa_shared(tc::smem_u32(spart), 0);
  for (int i = tid; i < kHeadRows * labels; i += kHeadThreads) {
    const int j = i / labels, l = i % labels;
    float s = 0.f;
#pragma unroll 8
    for (int c = 0; c < kHeadCols; ++c) s += pooled[j * kHeadCols + c] * swc[l * kHeadCols + c];
    tc::st_shared_cluster_s32(part0 + 4u * (uint32_t)((cb * kHeadRows + j) * kHeadMaxLabels + l),
                              __float_as_int(s));
  }
  tc::cluster_sync_all();
  if (tc::cluster_ctarank() != 0) return;
  for (int i = tid; i < kHeadRows * labels; i += kHeadThreads) {
    const int j = i / labels, l = i % labels;
    if (r0 + j >= rows) continue;
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < kHeadColBlocks; ++c) s += spart[(c * kHeadRows + j) * kHeadMaxLabels + l];
    logits[(int64_t)(r0 + j) * ld_logits + l] = s + __ldg(b_cls + l);
  }
}

}  // namespace gg

using namespace gg;

extern "C" int gg_cls_head(const void* hidden, int64_t ld_rows, const float* ln_gamma, const float* ln_beta,
                           float eps, const void* w_pre, const float* b_pre, const void* w_cls,
                           const float* b_cls, int32_t labels, float* logits, int64_t ld_logits, int32_t rows,
                           int32_t max_rows, const int32_t* count_dev, float* scratch, int32_t* arrivals,
                           void* stream) {
  (void)scratch;
  (void)arrivals;
  if (!hidden || !w_pre || !b_pre || !w_cls || !b_cls || !logits || rows < 0 ||
      rows > max_rows || (!ln_gamma) != (!ln_beta))
    return GG_ERR_INVALID_ARGUMENT;
  if (labels < 1 || labels > kHeadMaxLabels || ld_rows % 8 || ld_logits < labels) return GG_ERR_UNSUPPORTED;
  if (rows == 0) return GG_OK;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(cls_head_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kHeadSmemAll) !=
        cudaSuccess)
      return GG_ERR_CUDA;
    attr = true;
  }
  (void)max_rows;   // scratch / arrivals: kept in the ABI, unused since the cluster reduction
  const dim3 grid(kHeadColBlocks, (unsigned)((rows + kHeadRows - 1) / kHeadRows));
  if (launch_pdl(cls_head_kernel, grid, dim3(kHeadThreads), kHeadSmemAll, gg_stream(stream),
                 reinterpret_cast<const __nv_bfloat16*>(hidden), ld_rows, ln_gamma, ln_beta, eps,
                 reinterpret_cast<const __nv_bfloat16*>(w_pre), b_pre, reinterpret_cast<const __nv_bfloat16*>(w_cls),
                 b_cls, (int)labels, logits, ld_logits, (int)rows, count_dev) != cudaSuccess)
    return GG_ERR_CUDA;
  GG_LAUNCH_OK();
  return GG_OK;
}

extern "C" int64_t gg_cls_head_scratch_bytes(int32_t max_rows) {
  return (int64_t)kHeadColBlocks * max_rows * kHeadMaxLabels * 4;
}
