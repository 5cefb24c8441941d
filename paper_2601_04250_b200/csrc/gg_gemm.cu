// gg_gemm.cu — tcgen05/TMEM GEMM with TMA operand loads and fused epilogues.
//
//   D[M, N] = act( A[M, K] . B[N, K]^T + bias[N] (+ residual[M, N]) )     bf16 out
//
// A and B are bf16, K-contiguous (activations x nn.Linear weight layout), fp32
// accumulation in tensor memory.  One CTA computes a BM x BN tile:
//   warp 0      TMA producer (one elected lane), S-stage smem ring, mbarriers
//   warp 1      TMEM allocator + tcgen05.mma issuer (one elected lane)
//   warps 2..5  epilogue: tcgen05.ld -> bias/residual/activation -> bf16 stores
// The CTA is persistent over tiles (grid = #SMs); the accumulator is double
// buffered in TMEM so the epilogue of tile i overlaps the MMAs of tile i+1.
#include <cudaTypedefs.h>
#include <limits.h>
#include <stdio.h>

#include "gg_common.cuh"
#include "gg_kernels.h"
#include "gg_streamk.cuh"
#include "gg_tc.cuh"

namespace gg {
using namespace tc;

enum : int { ACT_NONE = 0, ACT_RELU = 1, ACT_GELU = 2 };

enum : int { OUT_BF16 = 0, OUT_F32 = 1, OUT_QKV_HEADS = 2 };

struct GemmEpilogue {
  void* D;
  int64_t ldd;
  const float* bias;               // [N] or null
  const __nv_bfloat16* residual;   // [M, ldr] or null
  int64_t ldr;
  int act;
  int out_mode;                    // OUT_*
  int seq_len;                     // OUT_QKV_HEADS: tokens per sequence (S)
  int heads;                       // OUT_QKV_HEADS: H (head dim fixed at 64)
  int64_t qkv_plane;               // OUT_QKV_HEADS: elements per Q/K/V^T plane (B*H*S*64)
  const int32_t* count;            // device item count (dynamic batch) or null
  int rows_per_item;               // M_eff = min(M, *count * rows_per_item)
  StreamK sk;                      // stream-K split of the (tile, k-block) space, or disabled
  int raster_n;                    // 1: N-fastest tile order (A larger than ~L2/2), else M-fastest
  long long* prof;                 // debug (GG_GEMM_PROF): per-pair issuer cycles / waits, or null
  int tma_out;                     // pair kernel: outputs (and residual) through smem + TMA
  int dbg_skip_epi;                // GG_GEMM_SKIP_EPI (probe): release accumulators without the epilogue
  // tile-level dependencies (gg_dep, pair kernel): 128-row unit counters
  const int* dep_wait;
  int dep_need;
  int* dep_signal;
  int* dep_go;
  int* dep_tiles;                  // dynamic tile counter (zeroed per chain) or null: static schedule
  int dep_dbg;                     // GG_DEP_DBG probe bits (1 no producer proxy fence, 2 relaxed poll,
                                   // 4 no signal fences)
  // LayerNorm folding (pair kernel, TMA epilogue; see gg_gemm_ln):
  const float2* a_stats;           // row statistics partials of A (raw h rows), [a_parts][ln_ld]
  const float* a_colsum;           // [N] s_j = sum_k W'_jk (W' = W diag(gamma))
  const float2* r_stats;           // row statistics partials of the residual rows
  const float* r_gamma;            // [ln_width] gamma / beta of the residual's LayerNorm
  const float* r_beta;
  float2* out_stats;               // this GEMM's output row partials, [N / 128][ln_ld]
  int a_parts, r_parts, ln_width;
  int64_t ln_ld;                   // rows per partial plane (the GEMM's M)
  float eps;
};

// LayerNorm row statistics carried between kernels as partials: one (mean_i,
// M2_i) per 128 columns of a row (one epilogue warp's slice), merged with
// Chan's formula by the consumer: mean = avg(mean_i), M2 = sum M2_i +
// 128 sum (mean_i - mean)^2, var = M2 / width (biased, like torch).
__device__ __forceinline__ void ln_row_params(const float2* st, int parts, int64_t ld, int64_t row,
                                              int width, float eps, float& scale, float& shift) {
  float m[8], q[8];
  float mean = 0.0f;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    if (i < parts) {
      const float2 v = __ldcg(st + (int64_t)i * ld + row);   // L2: written by a live producer
      m[i] = v.x;
      q[i] = v.y;
      mean += v.x;
    }
  }
  mean /= (float)parts;
  float m2 = 0.0f;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    if (i < parts) {
      const float d = m[i] - mean;
      m2 += q[i] + 128.0f * d * d;
    }
  }
  const float rstd = rsqrtf(m2 / (float)width + eps);
  scale = rstd;
  shift = -mean * rstd;
}

constexpr int kBK = 64;            // 64 bf16 = 128 B = one swizzle row

__device__ __forceinline__ long long gtimer_ns() {   // GG_GEMM_PROF timeline stamps
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// 8 epilogue warps: two per TMEM lane quarter, each draining half of the tile's
// columns, so bias/GELU/residual math keeps pace with the MMA of the next tile.
constexpr int kEpiWarps = 8;
constexpr int kThreads = 64 + 32 * kEpiWarps;

template <int BM, int BN, int STAGES>
struct GemmSmem {
  static constexpr int A_BYTES = BM * kBK * 2;
  static constexpr int B_BYTES = BN * kBK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int BAR_OFF = STAGES * STAGE_BYTES;
  static constexpr int TOTAL = BAR_OFF + 256 + 1024;  // + barriers + alignment slack
};

// Fused epilogue of one thread's 32 consecutive accumulator columns of one row:
// bias, residual, activation and the output layout.
__device__ __forceinline__ void epi_chunk(const GemmEpilogue& ep, int row, int col0, float (&v)[32],
                                          const uint4* res_pre = nullptr,
                                          const float* bias_smem = nullptr) {
  if (ep.bias) {
    const float* bsrc = bias_smem ? bias_smem : ep.bias;
#pragma unroll
    for (int i = 0; i < 32; i += 4) {
      float4 b = *reinterpret_cast<const float4*>(bsrc + col0 + i);
      v[i] += b.x; v[i + 1] += b.y; v[i + 2] += b.z; v[i + 3] += b.w;
    }
  }
  if (ep.residual) {
    const uint4* rp = reinterpret_cast<const uint4*>(ep.residual + (int64_t)row * ep.ldr + col0);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint4 u = res_pre ? res_pre[q] : rp[q];
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float2 f = __bfloat1622float2(h[e]);
        v[q * 8 + 2 * e] += f.x;
        v[q * 8 + 2 * e + 1] += f.y;
      }
    }
  }
  if (ep.act == ACT_RELU) {
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = fmaxf(v[i], 0.0f);
  } else if (ep.act == ACT_GELU) {
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = gelu_erf(v[i]);
  }
  if (ep.out_mode == OUT_F32) {
    float4* dp = reinterpret_cast<float4*>(reinterpret_cast<float*>(ep.D) + (int64_t)row * ep.ldd + col0);
#pragma unroll
    for (int q = 0; q < 8; ++q) dp[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    return;
  }
  __nv_bfloat16* dst;
  if (ep.out_mode == OUT_QKV_HEADS) {
    // [M, 3*H*64] -> Q (pre-scaled by 1/sqrt(64), exact), K as [B,H,S,64]; V^T as [B,H,64,S]
    const int hd = ep.heads * 64;
    const int which = col0 / hd, h = (col0 % hd) / 64, d0 = col0 % 64;
    const int b = row / ep.seq_len, s_ = row % ep.seq_len;
    __nv_bfloat16* plane = reinterpret_cast<__nv_bfloat16*>(ep.D) + which * ep.qkv_plane;
    const int64_t bh = (int64_t)b * ep.heads + h;
    if (which == 2) {
#pragma unroll
      for (int i = 0; i < 32; ++i)
        plane[(bh * 64 + d0 + i) * ep.seq_len + s_] = __float2bfloat16_rn(v[i]);
      return;
    }
    if (which == 0) {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] *= 0.125f;
    }
    dst = plane + (bh * ep.seq_len + s_) * 64 + d0;
  } else {
    dst = reinterpret_cast<__nv_bfloat16*>(ep.D) + (int64_t)row * ep.ldd + col0;
  }
  uint4* dp = reinterpret_cast<uint4*>(dst);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint4 u;
    u.x = pack_bf16(v[q * 8 + 0], v[q * 8 + 1]);
    u.y = pack_bf16(v[q * 8 + 2], v[q * 8 + 3]);
    u.z = pack_bf16(v[q * 8 + 4], v[q * 8 + 5]);
    u.w = pack_bf16(v[q * 8 + 6], v[q * 8 + 7]);
    dp[q] = u;
  }
}

template <int BM, int BN, int STAGES>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_bf16_tcgen05(const __grid_constant__ CUtensorMap map_a,
                      const __grid_constant__ CUtensorMap map_b, int M_max, int N, int K,
                      GemmEpilogue ep) {
  using L = GemmSmem<BM, BN, STAGES>;
  static_assert(BM == 128, "cta_group::1 tiles use all 128 TMEM lanes");
  static_assert(2 * BN <= 512, "two accumulators must fit TMEM");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_align1k(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::BAR_OFF);
  uint64_t* empty = full + STAGES;
  uint64_t* acc_full = empty + STAGES;     // [2]
  uint64_t* acc_empty = acc_full + 2;      // [2]
  uint32_t* tmem_base_smem = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  griddep_launch();   // the successor may begin its prologue as SMs free up
  const int num_kb = K / kBK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&acc_full[a], 1);
      mbar_init(&acc_empty[a], kEpiWarps);
    }
    fence_mbar_init();
    tma_prefetch(&map_a);
    tma_prefetch(&map_b);
  }
  if (warp == 1) tmem_alloc(tmem_base_smem, 2 * BN);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_base_smem;
  griddep_wait();   // operands, count and output follow the stream predecessor
  // dynamic batch: the admitted count is read on the device (no host round-trip)
  const int M = ep.count ? min(M_max, __ldg(ep.count) * ep.rows_per_item) : M_max;
  const int tiles_m = (M + BM - 1) / BM, tiles_n = (N + BN - 1) / BN;
  const int num_tiles = tiles_m * tiles_n;

  if (warp == 0) {
    // ===== TMA producer =====
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      SkSched sc(ep.sk.enabled, num_tiles, num_kb, blockIdx.x, gridDim.x);
      SkWork w;
      while (sc.next(w)) {
        // raster: M-fastest keeps the weight tile hot across consecutive CTAs; when
        // A outgrows the L2 (FFN-down: 100 MB) N-fastest makes the CTAs working at
        // once share A row blocks (read from HBM once, reused across the N tiles)
        const int tm = ep.raster_n ? w.tile / tiles_n : w.tile % tiles_m;
        const int tn = ep.raster_n ? w.tile % tiles_n : w.tile / tiles_m;
        for (int kb = w.kb0; kb < w.kb1; ++kb) {
          mbar_wait_sleep(&empty[s], ph ^ 1);
          uint8_t* sa = smem + s * L::STAGE_BYTES;
          uint8_t* sb = sa + L::A_BYTES;
          mbar_expect_tx(&full[s], L::STAGE_BYTES);
          tma_load_2d(sa, &map_a, &full[s], kb * kBK, tm * BM);
          tma_load_2d(sb, &map_b, &full[s], kb * kBK, tn * BN);
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===== MMA issuer: the warp runs the loop, one elected lane issues =====
    {
      constexpr uint32_t idesc = idesc_bf16_f32(BM, BN);
      int s = 0, t = 0;
      uint32_t ph = 0;
      const uint64_t a_desc0 = sdesc_k_sw128(smem_u32(smem));
      SkSched sc(ep.sk.enabled, num_tiles, num_kb, blockIdx.x, gridDim.x);
      SkWork w;
      for (; sc.next(w); ++t) {
        const int acc = t & 1;
        const uint32_t use = t >> 1;
        mbar_wait(&acc_empty[acc], (use & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = w.kb0; kb < w.kb1; ++kb) {   // lean chain: incremental ring / descriptors
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint64_t ad = a_desc0 + (uint64_t)s * (uint64_t)(L::STAGE_BYTES >> 4);
          const uint64_t bd = ad + (uint64_t)(L::A_BYTES >> 4);
          if (elect_one_sync()) {
#pragma unroll
            for (int kk = 0; kk < kBK / 16; ++kk)
              umma_bf16(d_tmem, ad + (uint64_t)(kk * 2), bd + (uint64_t)(kk * 2), idesc,
                        (kb != w.kb0 || kk != 0));
            umma_commit(&empty[s]);
          }
          __syncwarp();
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
        if (elect_one_sync()) umma_commit(&acc_full[acc]);
        __syncwarp();
      }
    }
  } else {
    // ===== epilogue warps =====
    const int quarter = warp & 3;  // TMEM lane quarter this warp may access
    const int half = (warp - 2) >> 2;  // which half of the columns
    int t = 0;
    SkSched sc(ep.sk.enabled, num_tiles, num_kb, blockIdx.x, gridDim.x);
    SkWork w;
    for (; sc.next(w); ++t) {
      const int tm = ep.raster_n ? w.tile / tiles_n : w.tile % tiles_m;
      const int tn = ep.raster_n ? w.tile % tiles_n : w.tile / tiles_m;
      const int acc = t & 1;
      const uint32_t use = t >> 1;
      mbar_wait_sleep(&acc_full[acc], use & 1);
      tc_fence_after();
      const uint32_t tacc = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * BN;
      // stream-K: a tile cut between CTAs is reduced by its last arriving segment
      const bool partial = w.kb0 != 0 || w.kb1 != num_kb;
      SkFix fx;
      if (partial) {
        auto load32 = [&](int c, float (&v)[32]) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(tacc + half * (BN / 2) + c, r);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
        };
        if (!sk_arrive<BN / 2>(ep.sk, sc, w, warp - 2, kEpiWarps, lane, fx, load32)) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&acc_empty[acc]);
          continue;
        }
      }
      const int row = tm * BM + quarter * 32 + lane;
      const bool row_ok = row < M;
#pragma unroll 1
      for (int c = half * (BN / 2); c < (half + 1) * (BN / 2); c += 32) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(tacc + c, r);
        tmem_ld_wait();
        const int col0 = tn * BN + c;
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
        if (partial) sk_sum<BN / 2>(ep.sk, sc, w, warp - 2, kEpiWarps, lane, fx, c - half * (BN / 2), v);
        if (!row_ok || col0 >= N) continue;
        epi_chunk(ep, row, col0, v);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[acc]);
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 2 * BN);
  }
}

// ---------------------------------------------------------------------------
// Host side: tensor-map encoding through the driver entry point (no -lcuda).
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

static int get_encoder() {
  if (g_encode) return GG_OK;
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !fn)
    return GG_ERR_CUDA;
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  return GG_OK;
}

// 2-D bf16 K-major operand [rows, cols] with row pitch ld (elements); box =
// [64 cols (128 B), box_rows], 128-byte swizzle, OOB -> 0.
int make_map_2d(CUtensorMap* map, const void* ptr, int64_t rows, int64_t cols, int64_t ld,
                int box_rows) {
  if (get_encoder() != GG_OK) return GG_ERR_CUDA;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? GG_OK : GG_ERR_INVALID_ARGUMENT;
}

// Stream-K workspace, one per device (see gg_streamk.cuh).
constexpr int64_t kSkWsFloats = 12LL << 20;      // 48 MB of fp32 partial regions
constexpr int64_t kSkCounters = 512LL << 10;     // 2 MB of (arrival, ready) counters
static StreamK g_sk[64];

static bool sk_alloc(int dev) {
  StreamK& s = g_sk[dev];
  if (s.ws) return true;
  float* ws = nullptr;
  int* cnt = nullptr;
  if (cudaMalloc(&ws, kSkWsFloats * sizeof(float)) != cudaSuccess) return false;
  if (cudaMalloc(&cnt, kSkCounters * sizeof(int)) != cudaSuccess ||
      cudaMemset(cnt, 0, kSkCounters * sizeof(int)) != cudaSuccess ||
      cudaDeviceSynchronize() != cudaSuccess) {
    cudaFree(ws);
    return false;
  }
  s.ws = ws;
  s.cnt = cnt;
  return true;
}

StreamK streamk_workspace(cudaStream_t stream, int64_t ws_floats, int64_t counters, bool& ok) {
  int dev = 0;
  cudaGetDevice(&dev);
  ok = false;
  StreamK none{nullptr, nullptr, 0};
  if (dev < 0 || dev >= 64 || ws_floats > kSkWsFloats || counters > kSkCounters) return none;
  if (!g_sk[dev].ws) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(stream, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone)
      return none;   // no allocation inside a graph capture: run data-parallel
    if (!sk_alloc(dev)) return none;
  }
  ok = true;
  StreamK s = g_sk[dev];
  s.enabled = 1;
  return s;
}

// Stream-K or data-parallel for `tiles` tiles of `nkb` k-blocks on `sms` SMs
// (policy -1): stream-K when it removes a partly empty last wave (fixup ~2
// k-blocks per CTA).  GG_STREAMK / gg_streamk_mode: 0 never (default), 1 force,
// -1 by this wave model.
static int g_sk_mode = -2;
static int sk_mode() {
  // default OFF: measured slower than data-parallel tiles at every DistilBERT /
  // ResNet shape (the fixup reads of the partial regions are latency-bound)
  if (g_sk_mode == -2) g_sk_mode = getenv("GG_STREAMK") ? atoi(getenv("GG_STREAMK")) : 0;
  return g_sk_mode;
}

bool streamk_wanted(int64_t tiles, int64_t nkb, int sms) {
  const int mode = sk_mode();
  if (mode == 0) return false;
  const int64_t T = tiles * nkb;
  if (mode == 1) return T >= 2 * sms;
  const double dp = (double)((tiles + sms - 1) / sms) * nkb;
  const double sk = (double)T / sms + 2.0;
  return T / sms >= 4 && sk < 0.93 * dp;
}

// [rows, cols] bf16 with row pitch ld (elements); box 32 x 32, 64-byte swizzle:
// the pair GEMM's epilogue staging boxes (TMA store of outputs, TMA load of residuals).
static int make_map_box32(CUtensorMap* map, const void* ptr, int64_t rows, int64_t cols, int64_t ld) {
  if (get_encoder() != GG_OK) return GG_ERR_CUDA;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides,
                        box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? GG_OK : GG_ERR_INVALID_ARGUMENT;
}

static int g_num_sms = 0;
static int g_sm_reserve = 0;   // gg_set_sm_reserve: SMs persistent grids leave free
static int device_sms() {
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return g_num_sms;
}
int num_sms() { return device_sms() - g_sm_reserve; }

template <int BM, int BN, int STAGES>
static int launch_gemm(const CUtensorMap& ma, const CUtensorMap& mb, int M, int N, int K,
                       GemmEpilogue ep, cudaStream_t s, int max_ctas) {
  using L = GemmSmem<BM, BN, STAGES>;
  auto kern = gemm_bf16_tcgen05<BM, BN, STAGES>;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::TOTAL) != cudaSuccess)
      return GG_ERR_CUDA;
    attr = true;
  }
  const int tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
  int grid = tiles < num_sms() ? tiles : num_sms();
  if (max_ctas > 0 && grid > max_ctas) grid = max_ctas;
  ep.sk = StreamK{nullptr, nullptr, 0};
  if (max_ctas <= 0 && streamk_wanted(tiles, K / kBK, num_sms())) {
    bool ok = false;
    const int g = num_sms();
    StreamK sk = streamk_workspace(s, (int64_t)g * 2 * BM * BN, (int64_t)tiles * kEpiWarps * 2, ok);
    if (ok) {
      ep.sk = sk;
      grid = g;
    }
  }
  if (launch_pdl(kern, dim3(grid), dim3(kThreads), (size_t)L::TOTAL, s, ma, mb, M, N, K, ep) != cudaSuccess)
    return GG_ERR_CUDA;
  GG_LAUNCH_OK();
  return GG_OK;
}


// ---------------------------------------------------------------------------
// CTA-pair GEMM (cluster of 2, cta_group::2): the pair computes a 256 x 256
// tile; each CTA stages its own 128 rows of A and its half (128 rows) of B per
// k-block, the leader issues M = 256, N = 256 MMAs that read both CTAs' smem and
// accumulate each CTA's 128 rows into its own TMEM.  Per SM that is 32 KB of
// operand ingress per 512 MMA cycles (64 B/cycle) instead of 48 KB (96 B/cycle)
// for a 128 x 256 single-CTA tile: the single-CTA kernel is bounded by the
// L2 -> SM operand bandwidth (~43 B/cycle/SM measured) at ~45 % of the tensor
// peak, the pair kernel at ~66 %.
//   warp 0     TMA producer in both CTAs (complete_tx on the leader's barrier)
//   warp 1     TMEM allocator (both CTAs) + MMA issuer (leader only)
//   warps 2-9  epilogue in both CTAs (their own 128 rows), release to the leader
constexpr int kPairBN = 256;
constexpr int kPairMaxN = 4096;   // bias staged in smem
constexpr int kPairAuxFloats = 3072;   // LN folding: s_j (N <= 3072) or gamma | beta (width <= 1536)

// Compile-time epilogue kinds of the pair kernel: the flags that shape the
// epilogue's instruction stream are template parameters (no per-chunk runtime
// branches); bias, ReLU, the residual LayerNorm and output statistics stay
// runtime flags (uniform branches, residual kernels only).
enum : int { EK_ALN = 1, EK_GELU = 2, EK_RES = 4, EK_QKV = 8 };

// EW epilogue warps (8 or 16): warp w drains TMEM lane quarter w % 4 and one of
// EW / 4 column parts of the tile (128 or 64 columns = 4 or 2 chunks of 32).
// NBUF 2 KB staging boxes per epilogue warp (residual kernels: 2, the next
// chunk's residual lands while this one is computed; otherwise 1).
template <int STAGES, int EW, int NBUF, int EK>
struct PairCfg {
  static constexpr int kThreads = 96 + 32 * EW;   // + the tile-scheduler warp
  static constexpr int A_BYTES = 128 * kBK * 2, B_BYTES = 128 * kBK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int BAR_OFF = STAGES * STAGE_BYTES;                  // barriers, tile ring, TMEM slot
  static constexpr int BAR_BYTES = 8 * (2 * STAGES + 4 + NBUF * EW + 12 + 8) + 4 * 4 + 4;
  static constexpr int BIAS_OFF = BAR_OFF + ((BAR_BYTES + 127) & ~127);  // [kPairMaxN] fp32
  static constexpr int STG_OFF = (BIAS_OFF + kPairMaxN * 4 + 1023) & ~1023;
  static constexpr int AUX_OFF = STG_OFF + EW * NBUF * 2048;           // [kPairAuxFloats] fp32
  static constexpr int SMEM = AUX_OFF + kPairAuxFloats * 4 + 1024;       // + alignment slack
  static_assert(SMEM <= 232448, "pair GEMM shared memory");
  static_assert(EW == 8 || EW == 16, "epilogue warps");
};

template <int STAGES, int EW, int NBUF, int EK>
__global__ void __launch_bounds__(96 + 32 * EW, 1)
    gemm_bf16_pair(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                   const __grid_constant__ CUtensorMap map_out, const __grid_constant__ CUtensorMap map_res,
                   int M_max, int N, int K, GemmEpilogue ep) {
  using C = PairCfg<STAGES, EW, NBUF, EK>;
  constexpr bool ALN = EK & EK_ALN, GELU = EK & EK_GELU, RES = EK & EK_RES, QKV = EK & EK_QKV;
  constexpr int PARTS = EW / 4, CW = kPairBN / PARTS, NCH = CW / 32;
  static_assert(!RES || NBUF >= 2, "residual boxes need a second staging buffer");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // stay in the shared window (LDS / STS, not generic LD / ST): offset the
  // array itself instead of round-tripping the pointer through an integer
  const uint32_t raw_u32 = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_u32 + 1023u) & ~1023u) - raw_u32);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t* empty = full + STAGES;
  uint64_t* acc_full = empty + STAGES;     // [2]
  uint64_t* acc_empty = acc_full + 2;      // [2] (the leader's counts both CTAs' epilogues)
  uint64_t* res_full = acc_empty + 2;      // [EW warps][NBUF buffers]: residual boxes landed
  uint64_t* tile_full = res_full + NBUF * EW;   // [4] dynamic schedule: tile index published
  uint64_t* tile_empty = tile_full + 4;         // [4] (leader) every reader of the slot is done
  uint64_t* tile_took = tile_empty + 4;         // [4] (leader) its producer started this slot's tile
  uint64_t* dep_ok = tile_took + 4;             // [8] the producer acquired this tile's unit
  int* tile_ring = reinterpret_cast<int*>(dep_ok + 8);   // [4] tile indices
  uint32_t* tmem_base_smem = reinterpret_cast<uint32_t*>(tile_ring + 4);
  float* bias_s = reinterpret_cast<float*>(smem + C::BIAS_OFF);   // [N] (N <= kPairMaxN)
  // per epilogue warp: NBUF 2 KB staging buffers = the SWIZZLE_64B image of a
  // 32 x 32 bf16 box (output for the TMA store, residual from a TMA load)
  uint8_t* stg_base = smem + C::STG_OFF;
  // LayerNorm folding: column sums s_j [N] (A side) or gamma | beta (residual side)
  float* aux_s = reinterpret_cast<float*>(smem + C::AUX_OFF);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  if (ep.prof && threadIdx.x == 0 && rank == 0) {
    ep.prof[pair * 8 + 4] = gtimer_ns();
    ep.prof[2048 + pair * 2] = clock64();
  }
  griddep_launch();
  const int num_kb = K / kBK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&acc_full[a], 1);
      mbar_init(&acc_empty[a], 2);   // one elected arrive per CTA of the pair
    }
    for (int i = 0; i < NBUF * EW; ++i) mbar_init(&res_full[i], 1);
    for (int i = 0; i < 4; ++i) {
      mbar_init(&tile_full[i], 1);
      // readers: both producers, the leader's MMA warp, both CTAs' epilogue warps
      mbar_init(&tile_empty[i], 3 + 2 * EW);
      mbar_init(&tile_took[i], 1);
    }
    for (int i = 0; i < 8; ++i) mbar_init(&dep_ok[i], 1);
    fence_mbar_init();
    tma_prefetch(&map_a);
    tma_prefetch(&map_b);
    tma_prefetch(&map_out);
    if (RES || QKV) tma_prefetch(&map_res);
  }
  if (warp == 1) tmem_alloc_pair(tmem_base_smem, 2 * kPairBN);
  tc_fence_before();
  cluster_sync_all();   // barriers of both CTAs initialised before any remote arrive / TMA
  tc_fence_after();
  const uint32_t tmem_base = *tmem_base_smem;
  int* cnt_slot = reinterpret_cast<int*>(tmem_base_smem + 1);
  if (ep.dep_wait) {
    // tile-level dependencies: no grid-wide wait; the batch count is read once
    // the chain's first kernel has passed its grid-wide wait
    if (threadIdx.x == 0) {
      dep_wait_geq(ep.dep_go, 1);
      *cnt_slot = ep.count ? ld_relaxed_gpu(ep.count) : 0;
    }
    __syncthreads();
  } else {
    griddep_wait();
    if (ep.dep_go && blockIdx.x == 0 && threadIdx.x == 0) dep_set(ep.dep_go, 1);
    if (threadIdx.x == 0) *cnt_slot = ep.count ? __ldg(ep.count) : 0;
    __syncthreads();
  }
  if (ep.prof && threadIdx.x == 0 && rank == 0) ep.prof[pair * 8 + 5] = gtimer_ns();
  const int M = ep.count ? min(M_max, *cnt_slot * ep.rows_per_item) : M_max;
  const int tiles_m = (M + 255) / 256, tiles_n = N / kPairBN;
  const int num_tiles = tiles_m * tiles_n;
  // Tile schedule.  Static: tile = pair + i * npairs.  Dynamic (dep_tiles): the
  // leader's scheduler warp claims tiles from a global counter (pairs that start
  // early -- on SMs the previous kernel's last wave left idle -- take more tiles)
  // and publishes each index through a 4-slot ring in both CTAs' smem.  A warp of
  // its own: an mbarrier arrive releases, i.e. waits for the issuing thread's
  // outstanding atomics, so claims in the producer would stall its TMA issue.
  const bool dyn = ep.dep_tiles != nullptr;
  const uint32_t leader_tile_empty0 = mapa_shared(smem_u32(&tile_empty[0]), 0);
  // reader side: the i-th tile of this CTA (every role except the leader's producer)
  auto read_tile = [&](int i, bool release) -> int {
    if (!dyn) return pair + i * npairs;
    const int slot = i & 3;
    // the leader's own readers: CTA-scope acquire of the local producer's arrive;
    // the peer's: cluster-scope acquire of the leader's remote store + arrive
    if (rank == 0 || (ep.dep_dbg & 32)) mbar_wait(&tile_full[slot], (i >> 2) & 1);
    else mbar_wait_cluster(&tile_full[slot], (i >> 2) & 1);
    const int tile = tile_ring[slot];
    if (release && tile < num_tiles) {   // (control-dependent on the value read)
      if (rank == 0) mbar_arrive_relaxed(&tile_empty[slot]);
      else mbar_arrive_cluster_relaxed(leader_tile_empty0 + slot * 8);
    }
    return tile;
  };

  if (warp == 0) {
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      const uint32_t peer_full0 = mapa_shared(smem_u32(&tile_full[0]), 1);
      const uint32_t peer_ring0 = mapa_shared(smem_u32(&tile_ring[0]), 1);
      (void)peer_full0;
      (void)peer_ring0;
      for (int i = 0;; ++i) {
        const int tile = read_tile(i, true);
        if (tile >= num_tiles) break;
        if (dyn && rank == 0) mbar_arrive_relaxed(&tile_took[i & 3]);   // the scheduler may claim the next
        const int tm = ep.raster_n ? tile / tiles_n : tile % tiles_m;   // raster: see gemm_impl
        const int tn = ep.raster_n ? tile % tiles_n : tile / tiles_m;
        const int m0 = tm * 256 + rank * 128, n0 = tn * kPairBN + rank * 128;
        if (ep.dep_wait) {
          // this CTA's 128 A rows (unit 2 tm + rank) published by the producer; the
          // epilogue's residual / statistics reads follow through dep_ok (every
          // earlier kernel of the chain published before this unit's producer)
          if (m0 < M) {
            if (ep.dep_dbg & 2) {
              while (ld_relaxed_gpu(ep.dep_wait + tm * 2 + rank) < ep.dep_need) __nanosleep(100);
            } else {
              dep_wait_geq(ep.dep_wait + tm * 2 + rank, ep.dep_need);
            }
            if (!(ep.dep_dbg & 1)) fence_proxy_async_global();
          }
          mbar_arrive(&dep_ok[i & 7]);
        }
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait_sleep(&empty[s], ph ^ 1);
          uint8_t* sa = smem + s * C::STAGE_BYTES;
          if (rank == 0) mbar_expect_tx(&full[s], 2 * C::STAGE_BYTES);
          const uint32_t fb = mapa_shared(smem_u32(&full[s]), 0);
          tma_load_2d_pair(sa, &map_a, fb, kb * kBK, m0);
          tma_load_2d_pair(sa + C::A_BYTES, &map_b, fb, kb * kBK, n0);
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {   // leader: the warp runs the loop, one elected lane issues
      constexpr uint32_t idesc = idesc_bf16_f32(256, kPairBN);
      int s = 0, t = 0;
      uint32_t ph = 0;
      const uint64_t a_desc0 = sdesc_k_sw128(smem_u32(smem));
      long long w_acc = 0, w_full = 0;            // GG_GEMM_PROF: issuer wait cycles
      const long long t0 = ep.prof ? clock64() : 0;
      for (;; ++t) {
        int tile;
        if (dyn) {
          tile = 0;
          if (lane == 0) tile = read_tile(t, true);
          tile = __shfl_sync(0xffffffffu, tile, 0);
        } else {
          tile = read_tile(t, false);
        }
        if (tile >= num_tiles) break;
        const int acc = t & 1;
        if (ep.prof) {
          const long long a = clock64();
          mbar_wait(&acc_empty[acc], ((t >> 1) & 1) ^ 1);
          w_acc += clock64() - a;
        } else {
          mbar_wait(&acc_empty[acc], ((t >> 1) & 1) ^ 1);
        }
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * kPairBN;
        // lean per-k-block chain: ring position and descriptors advance incrementally
        for (int kb = 0; kb < num_kb; ++kb) {
          if (ep.prof) {
            const long long a = clock64();
            mbar_wait(&full[s], ph);
            w_full += clock64() - a;
          } else {
            mbar_wait(&full[s], ph);
          }
          tc_fence_after();
          const uint64_t ad = a_desc0 + (uint64_t)s * (uint64_t)(C::STAGE_BYTES >> 4);
          const uint64_t bd = ad + (uint64_t)(C::A_BYTES >> 4);
          if (elect_one_sync()) {
#pragma unroll
            for (int kk = 0; kk < kBK / 16; ++kk)
              umma_bf16_pair(d_tmem, ad + (uint64_t)(kk * 2), bd + (uint64_t)(kk * 2), idesc, (kb | kk) != 0);
            umma_commit_pair(&empty[s], 3);
          }
          __syncwarp();
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
        if (elect_one_sync()) umma_commit_pair(&acc_full[acc], 3);
        __syncwarp();
      }
      if (ep.prof && lane == 0) {
        ep.prof[pair * 8 + 0] = clock64() - t0;
        ep.prof[pair * 8 + 1] = w_acc;
        ep.prof[pair * 8 + 2] = w_full;
        ep.prof[pair * 8 + 3] = t;
        ep.prof[pair * 8 + 6] = gtimer_ns();
      }
    }
  } else if (warp == 2 + EW) {
    // ===== tile scheduler (leader, dynamic schedule): claim, publish to both CTAs
    if (dyn && rank == 0 && lane == 0) {
      const uint32_t peer_full0 = mapa_shared(smem_u32(&tile_full[0]), 1);
      const uint32_t peer_ring0 = mapa_shared(smem_u32(&tile_ring[0]), 1);
      for (int i = 0;; ++i) {
        const int slot = i & 3;
        // at most one claimed tile waits behind the one being loaded: claim tile i
        // once the producer has started tile i - 1 (pairs finish within ~a tile)
        if (i > 0) mbar_wait(&tile_took[(i - 1) & 3], ((i - 1) >> 2) & 1);
        mbar_wait(&tile_empty[slot], ((i >> 2) & 1) ^ 1);
        const int tile = atomicAdd(ep.dep_tiles, 1);
        tile_ring[slot] = tile;
        st_shared_cluster_s32(peer_ring0 + slot * 4, tile);
        mbar_arrive(&tile_full[slot]);
        mbar_arrive_cluster(peer_full0 + slot * 8);
        if (tile >= num_tiles) break;
      }
    }
  } else {
    // ===== epilogue warps: TMEM -> registers -> fused math -> SW64 smem box -> TMA store
    // A thread owns one accumulator row, so direct global stores / residual loads
    // would touch 32 rows (32 L1 wavefronts) per instruction; instead each warp
    // stages its 32 x 32 chunk in smem (SW64 image, conflict-free for row-per-lane
    // 16-B accesses) and moves it with one TMA store.  Residual boxes arrive by
    // TMA one chunk ahead.
    const int quarter = warp & 3;
    const int part = (warp - 2) >> 2;
    const int ew = warp - 2;
    const uint32_t leader_empty0 = mapa_shared(smem_u32(&acc_empty[0]), 0);
    // the bias vector once per CTA in smem (broadcast LDS instead of per-chunk LDG)
    if (ep.bias)
      for (int i = threadIdx.x - 64; i < N; i += 32 * EW) bias_s[i] = __ldg(ep.bias + i);
    if (ALN)
      for (int i = threadIdx.x - 64; i < N; i += 32 * EW) aux_s[i] = __ldg(ep.a_colsum + i);
    if (RES && ep.r_stats)
      for (int i = threadIdx.x - 64; i < ep.ln_width; i += 32 * EW) {
        aux_s[i] = __ldg(ep.r_gamma + i);
        aux_s[ep.ln_width + i] = __ldg(ep.r_beta + i);
      }
    asm volatile("bar.sync 1, %0;" ::"n"(32 * EW) : "memory");
    uint8_t* stg = stg_base + ew * (NBUF * 2048);
    uint64_t* rb = res_full + ew * NBUF;
    uint32_t rph = 0;   // parity bit per staging buffer
    const int sw = (lane >> 1) & 3;
    const bool has_bias = ep.bias != nullptr;
    int prev_unit = -1;   // unit of the previous tile, published one tile late
    int t = 0;
    for (;; ++t) {
      int tile;
      if (dyn) {
        tile = 0;
        if (lane == 0) tile = read_tile(t, true);
        tile = __shfl_sync(0xffffffffu, tile, 0);
      } else {
        tile = read_tile(t, false);
      }
      if (tile >= num_tiles) break;
      const int tm = ep.raster_n ? tile / tiles_n : tile % tiles_m;
      const int tn = ep.raster_n ? tile % tiles_n : tile / tiles_m;
      const int acc = t & 1;
      const int row0 = tm * 256 + rank * 128 + quarter * 32;   // this warp's 32 rows
      const int colw = tn * kPairBN + part * CW;                 // this warp's CW columns
      const bool rows_ok = row0 < M && !ep.dbg_skip_epi;
      const int unit = tm * 2 + (int)rank;
      if ((ALN || RES) && ep.dep_wait) {
        // the residual / statistics rows come from the producer or earlier kernels
        // of the chain: the local producer acquired this unit (its arrive releases
        // at CTA scope; the producer is < 8 tiles ahead: 2 TMEM buffers + its ring)
        mbar_wait(&dep_ok[t & 7], (t >> 3) & 1);
        if (RES && lane == 0) fence_proxy_async_global();
      }
      if (RES && rows_ok && lane == 0) {   // residual of chunk 0
        bulk_wait_read<0>();
        mbar_expect_tx(&rb[0], 2048);
        tma_load_2d(stg, &map_res, &rb[0], colw, row0);
      }
      // LayerNorm folding: this lane's row (row0 + lane) affine parameters
      float a_sc = 1.0f, a_sh = 0.0f, r_sc = 1.0f, r_sh = 0.0f;
      if (ALN && rows_ok)
        ln_row_params(ep.a_stats, ep.a_parts, ep.ln_ld, row0 + lane, ep.ln_width, ep.eps, a_sc, a_sh);
      if (RES && rows_ok && ep.r_stats)
        ln_row_params(ep.r_stats, ep.r_parts, ep.ln_ld, row0 + lane, ep.ln_width, ep.eps, r_sc, r_sh);
      float st_k = 0.0f, st_s1 = 0.0f, st_s2 = 0.0f;   // output row partial (shifted sums)
      int ngroups = 0;                                   // bulk store groups committed for this tile
      mbar_wait_sleep(&acc_full[acc], (t >> 1) & 1);
      tc_fence_after();
      const uint32_t tacc = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * kPairBN + part * CW;
#pragma unroll 1
      for (int c = 0; c < NCH; ++c) {
        const int b = NBUF == 1 ? 0 : (c & 1);
        uint8_t* buf = stg + b * 2048;
        if (RES && rows_ok && lane == 0 && c + 1 < NCH) {
          // next chunk's residual into the other buffer once its last store has read it
          bulk_wait_read<0>();
          mbar_expect_tx(&rb[b ^ 1], 2048);
          tma_load_2d(stg + (b ^ 1) * 2048, &map_res, &rb[b ^ 1], colw + 32 * (c + 1), row0);
        }
        uint32_t r[32];
        tmem_ld_32x32b_x32(tacc + 32 * c, r);
        tmem_ld_wait();
        if (!rows_ok) continue;
        const int col0 = colw + 32 * c;
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
        if (ALN) {   // LN(h) W^T + b = rstd (h W'^T) + (c_j - rstd mean s_j)
          const uint64_t sc2 = f2_pack(a_sc, a_sc), sh2 = f2_pack(a_sh, a_sh);
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            const float4 sj = *reinterpret_cast<const float4*>(aux_s + col0 + i);
            const float4 cj = *reinterpret_cast<const float4*>(bias_s + col0 + i);
            const uint64_t t0 = f2_fma(sh2, f2_pack(sj.x, sj.y), f2_pack(cj.x, cj.y));
            const uint64_t t1 = f2_fma(sh2, f2_pack(sj.z, sj.w), f2_pack(cj.z, cj.w));
            f2_unpack(f2_fma(sc2, f2_pack(v[i], v[i + 1]), t0), v[i], v[i + 1]);
            f2_unpack(f2_fma(sc2, f2_pack(v[i + 2], v[i + 3]), t1), v[i + 2], v[i + 3]);
          }
        } else if (has_bias) {
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            const float4 bb = *reinterpret_cast<const float4*>(bias_s + col0 + i);
            f2_unpack(f2_add(f2_pack(v[i], v[i + 1]), f2_pack(bb.x, bb.y)), v[i], v[i + 1]);
            f2_unpack(f2_add(f2_pack(v[i + 2], v[i + 3]), f2_pack(bb.z, bb.w)), v[i + 2], v[i + 3]);
          }
        }
        uint4* myrow = reinterpret_cast<uint4*>(buf + lane * 64);
        if (RES) {
          mbar_wait(&rb[b], (rph >> b) & 1u);
          rph ^= 1u << b;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint4 u = myrow[q ^ sw];
            const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&u);
            float rr[8];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 f = __bfloat1622float2(h2[e]);
              rr[2 * e] = f.x;
              rr[2 * e + 1] = f.y;
            }
            if (ep.r_stats) {   // residual = LayerNorm(raw h) on the fly
              const int cc = col0 + q * 8;
              const float4 g0 = *reinterpret_cast<const float4*>(aux_s + cc);
              const float4 g1 = *reinterpret_cast<const float4*>(aux_s + cc + 4);
              const float4 b0 = *reinterpret_cast<const float4*>(aux_s + ep.ln_width + cc);
              const float4 b1 = *reinterpret_cast<const float4*>(aux_s + ep.ln_width + cc + 4);
              const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
              const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
              const uint64_t sc2 = f2_pack(r_sc, r_sc), sh2 = f2_pack(r_sh, r_sh);
#pragma unroll
              for (int e = 0; e < 8; e += 2) {
                const uint64_t nrm = f2_fma(f2_pack(rr[e], rr[e + 1]), sc2, sh2);
                f2_unpack(f2_fma(nrm, f2_pack(gg[e], gg[e + 1]), f2_pack(bb[e], bb[e + 1])), rr[e],
                          rr[e + 1]);
              }
            }
#pragma unroll
            for (int e = 0; e < 8; e += 2)
              f2_unpack(f2_add(f2_pack(v[q * 8 + e], v[q * 8 + e + 1]), f2_pack(rr[e], rr[e + 1])),
                        v[q * 8 + e], v[q * 8 + e + 1]);
          }
        }
        if (GELU) {
#pragma unroll
          for (int i = 0; i < 32; i += 2) gelu_erf2(v[i], v[i + 1]);
        } else if (ep.act == ACT_RELU) {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = fmaxf(v[i], 0.0f);
        }
        int gx = col0, gy = row0;
        bool vt = false;   // QKV: this chunk is V, stored transposed
        if (QKV) {
          // Q (x 1/sqrt(64)) and K boxes into their [B, H, S, 64] planes; V^T boxes
          // (32 d x 32 s, transposed in the staging tile) into the [B, H, 64, S] plane
          const int hd = ep.heads * 64;
          const int which = col0 / hd, hh = (col0 % hd) / 64;
          if (which == 2) {
            vt = true;
            gx = row0 % ep.seq_len;
            gy = (int)(((int64_t)(row0 / ep.seq_len) * ep.heads + hh) * 64 + col0 % 64);
          }
          if (which == 0) {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] *= 0.125f;
          }
          if (!vt) {
            gx = col0 % 64;
            gy = (int)((int64_t)which * (ep.qkv_plane / 64) +
                       ((int64_t)(row0 / ep.seq_len) * ep.heads + hh) * ep.seq_len + row0 % ep.seq_len);
          }
        }
        uint4 u[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          u[q].x = pack_bf16(v[q * 8 + 0], v[q * 8 + 1]);
          u[q].y = pack_bf16(v[q * 8 + 2], v[q * 8 + 3]);
          u[q].z = pack_bf16(v[q * 8 + 4], v[q * 8 + 5]);
          u[q].w = pack_bf16(v[q * 8 + 6], v[q * 8 + 7]);
        }
        if (!RES) {   // the store that last read this buffer (NBUF chunks ago) is done
          if (lane == 0) bulk_wait_read<NBUF - 1>();
          __syncwarp();
        }
        if (QKV && vt) {
          // staging row i = head dim d0 + i (64 B, SW64: 16-B chunk c at c ^ ((i >> 1) & 3)),
          // column = sequence position (this lane): 32 conflict-free 2-B stores per lane
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const int off = i * 64 + ((((lane >> 3) ^ (i >> 1)) & 3) << 4) + ((lane & 7) << 1);
            *reinterpret_cast<__nv_bfloat16*>(buf + off) = __float2bfloat16_rn(v[i]);
          }
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q) myrow[q ^ sw] = u[q];
        }
        if (RES && ep.out_stats) {   // row statistics of this chunk (shifted sums, fp32 values)
          if (c == 0) st_k = v[0];
          const uint64_t nk = f2_pack(-st_k, -st_k);
          uint64_t s1 = f2_pack(0.0f, 0.0f), s2 = f2_pack(0.0f, 0.0f);
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            const uint64_t d = f2_add(f2_pack(v[i], v[i + 1]), nk);
            s1 = f2_add(s1, d);
            s2 = f2_fma(d, d, s2);
          }
          float a0, a1, c0, c1;
          f2_unpack(s1, a0, a1);
          f2_unpack(s2, c0, c1);
          st_s1 += a0 + a1;
          st_s2 += c0 + c1;
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_2d(QKV && vt ? &map_res : &map_out, buf, gx, gy);   // (QKV: map_res = the V^T plane)
          bulk_commit();
        }
        ++ngroups;
      }
      if (RES && ep.out_stats && rows_ok) {
        const float n = (float)CW;
        const float mi = st_k + st_s1 / n;
        const float m2 = fmaxf(st_s2 - st_s1 * st_s1 / n, 0.0f);
        ep.out_stats[(int64_t)(tn * PARTS + part) * ep.ln_ld + row0 + lane] = make_float2(mi, m2);
      }
      if (ep.dep_signal && lane == 0) {
        // the previous tile's stores (older groups than this tile's) are complete
        if (ngroups == 0) bulk_wait<0>();
        else if (ngroups == 1) bulk_wait<1>();
        else if (ngroups == 2) bulk_wait<2>();
        else if (ngroups == 3) bulk_wait<3>();
        else bulk_wait<4>();
        if (!(ep.dep_dbg & 4)) fence_proxy_async_global();
      }
      tc_fence_before();
      asm volatile("bar.sync 1, %0;" ::"n"(32 * EW) : "memory");
      if (threadIdx.x == 64) {
        if (rank == 0) mbar_arrive(&acc_empty[acc]);
        else mbar_arrive_cluster(leader_empty0 + acc * 8);
        // publish the previous tile (one tile late: its stores had this tile to land)
        if (ep.dep_signal && prev_unit >= 0) {
          // red.release: orders this thread's prior accesses and, cumulatively, the
          // CTA's output writes it observed through the barrier above
          if (ep.dep_dbg & 16) dep_signal_add(ep.dep_signal + prev_unit, 1);
          else dep_signal_add_nofence(ep.dep_signal + prev_unit, 1);
        }
      }
      prev_unit = tm * 256 + (int)rank * 128 < M ? unit : -1;
    }
    if (lane == 0) {
      bulk_wait<0>();
      fence_proxy_async_global();
    }
    if (ep.dep_signal) {
      asm volatile("bar.sync 1, %0;" ::"n"(32 * EW) : "memory");
      if (threadIdx.x == 64 && prev_unit >= 0) dep_signal_add_nofence(ep.dep_signal + prev_unit, 1);
    }
    if (ep.prof && threadIdx.x == 64 && rank == 0) {
      ep.prof[pair * 8 + 7] = gtimer_ns();
      ep.prof[2048 + pair * 2 + 1] = clock64();
    }
  }
  __syncthreads();
  cluster_sync_all();   // the peer's epilogue has released its last accumulator
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, 2 * kPairBN);
  }
}


// ---------------------------------------------------------------------------
// Fused FFN (DistilBERT lin1 + GELU -> lin2 + residual) as ONE persistent
// CTA-pair kernel.  The two GEMMs' tiles share one dynamic queue: lin1 tiles
// (256 x 256, K = 768, LayerNorm-folded A, exact-erf GELU) first, in row-block
// order, then lin2 tiles (256 x 256, K = 3072, LayerNorm'd residual, output row
// statistics).  A lin2 tile waits, in its producer, for the 12 lin1 tiles of
// its 128-row unit (per-unit counters: TMA stores complete -> proxy fence ->
// red.release; acquire -> proxy fence -> TMA loads), so pairs that run out of
// lin1 tiles start lin2 work at once: one kernel tail instead of two and the
// two GEMMs' partial last waves (10.38 + 2.59) merge.
constexpr int kFfnMaxUp = 3072;     // lin1 N (bias / column sums staged in smem)
constexpr int kFfnMaxDown = 768;    // lin2 N = LayerNorm width (bias, gamma | beta)
constexpr int kFfnStages = 5;
constexpr int kFfnEW = 8;
constexpr int kFfnThreads = 96 + 32 * kFfnEW;
struct FfnCfg {
  static constexpr int A_BYTES = 128 * kBK * 2, B_BYTES = 128 * kBK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int BAR_OFF = kFfnStages * STAGE_BYTES;
  static constexpr int BIAS0_OFF = BAR_OFF + 512;
  static constexpr int AUX0_OFF = BIAS0_OFF + kFfnMaxUp * 4;
  static constexpr int BIAS1_OFF = AUX0_OFF + kFfnMaxUp * 4;
  static constexpr int AUX1_OFF = BIAS1_OFF + kFfnMaxDown * 4;
  static constexpr int STG_OFF = (AUX1_OFF + 2 * kFfnMaxDown * 4 + 1023) & ~1023;
  static constexpr int SMEM = STG_OFF + kFfnEW * 2 * 2048 + 1024;
  static_assert(SMEM <= 232448, "fused FFN shared memory");
};

struct FfnArgs {
  int M_max;
  const int32_t* count;
  int rows_per_item;
  int n_up, n_down, k_up;           // lin1 N (= lin2 K), lin2 N (= lin1 K = LayerNorm width)
  const float* bias0;               // lin1 folded bias c_j
  const float* colsum0;             // lin1 column sums s_j of W' = W diag(gamma)
  const float2* a_stats;            // statistics partials of lin1's raw input rows
  const float* bias1;               // lin2 bias
  const float2* r_stats;            // residual rows' statistics partials (LayerNorm'd on the fly)
  const float* r_gamma;
  const float* r_beta;
  float2* out_stats;                // lin2 output rows' partials
  int parts;                        // partials per row (width / 128)
  int64_t ln_ld;
  float eps;
  int* ready;                       // [units] lin1 tiles published per 128-row unit (zeroed)
  int* tiles;                       // tile claim counter (zeroed)
  long long* prof;                  // GG_GEMM_PROF: per pair [issuer, acc wait, operand wait, tiles,
                                    //  lin2 dependency wait, lin1 tiles], or null
};

__global__ void __launch_bounds__(kFfnThreads, 1)
    gemm_ffn_pair(const __grid_constant__ CUtensorMap map_a0, const __grid_constant__ CUtensorMap map_b0,
                  const __grid_constant__ CUtensorMap map_o0, const __grid_constant__ CUtensorMap map_a1,
                  const __grid_constant__ CUtensorMap map_b1, const __grid_constant__ CUtensorMap map_o1,
                  const __grid_constant__ CUtensorMap map_r1, FfnArgs f) {
  using Cf = FfnCfg;
  constexpr int EW = kFfnEW, STAGES = kFfnStages, PARTS = EW / 4, CW = kPairBN / PARTS, NCH = CW / 32;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_align1k(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cf::BAR_OFF);
  uint64_t* empty = full + STAGES;
  uint64_t* acc_full = empty + STAGES;     // [2]
  uint64_t* acc_empty = acc_full + 2;      // [2]
  uint64_t* res_full = acc_empty + 2;      // [EW][2]
  uint64_t* tile_full = res_full + 2 * EW; // [4]
  uint64_t* tile_empty = tile_full + 4;    // [4]
  uint64_t* tile_took = tile_empty + 4;    // [4]
  int* tile_ring = reinterpret_cast<int*>(tile_took + 4);
  uint32_t* tmem_base_smem = reinterpret_cast<uint32_t*>(tile_ring + 4);
  int* cnt_slot = reinterpret_cast<int*>(tmem_base_smem + 1);
  float* bias0_s = reinterpret_cast<float*>(smem + Cf::BIAS0_OFF);
  float* aux0_s = reinterpret_cast<float*>(smem + Cf::AUX0_OFF);
  float* bias1_s = reinterpret_cast<float*>(smem + Cf::BIAS1_OFF);
  float* aux1_s = reinterpret_cast<float*>(smem + Cf::AUX1_OFF);
  uint8_t* stg_base = smem + Cf::STG_OFF;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  griddep_launch();
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&acc_full[a], 1);
      mbar_init(&acc_empty[a], 2);
    }
    for (int i = 0; i < 2 * EW; ++i) mbar_init(&res_full[i], 1);
    for (int i = 0; i < 4; ++i) {
      mbar_init(&tile_full[i], 1);
      mbar_init(&tile_empty[i], 3 + 2 * EW);
      mbar_init(&tile_took[i], 1);
    }
    fence_mbar_init();
    tma_prefetch(&map_a0);
    tma_prefetch(&map_b0);
    tma_prefetch(&map_o0);
    tma_prefetch(&map_a1);
    tma_prefetch(&map_b1);
    tma_prefetch(&map_o1);
    tma_prefetch(&map_r1);
  }
  if (warp == 1) tmem_alloc_pair(tmem_base_smem, 2 * kPairBN);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_base_smem;
  griddep_wait();   // lin1's input rows, statistics and the count follow the predecessor
  if (threadIdx.x == 0) *cnt_slot = f.count ? __ldg(f.count) : 0;
  __syncthreads();
  const int M = f.count ? min(f.M_max, *cnt_slot * f.rows_per_item) : f.M_max;
  const int tiles_m = (M + 255) / 256;
  const int tn0 = f.n_up / kPairBN, tn1 = f.n_down / kPairBN;
  const int T0 = tiles_m * tn0, num_tiles = T0 + tiles_m * tn1;
  const int kb0 = f.k_up / kBK, kb1 = f.n_up / kBK;
  const uint32_t leader_tile_empty0 = mapa_shared(smem_u32(&tile_empty[0]), 0);
  auto read_tile = [&](int i, bool release) -> int {
    const int slot = i & 3;
    if (rank == 0) mbar_wait(&tile_full[slot], (i >> 2) & 1);
    else mbar_wait_cluster(&tile_full[slot], (i >> 2) & 1);
    const int tile = tile_ring[slot];
    if (release && tile < num_tiles) {
      if (rank == 0) mbar_arrive_relaxed(&tile_empty[slot]);
      else mbar_arrive_cluster_relaxed(leader_tile_empty0 + slot * 8);
    }
    return tile;
  };

  if (warp == 0) {
    // ===== TMA producer (both CTAs)
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      long long wdep = 0;
      int nup = 0;
      for (int i = 0;; ++i) {
        const int tile = read_tile(i, true);
        if (tile >= num_tiles) break;
        if (rank == 0) mbar_arrive_relaxed(&tile_took[i & 3]);
        const bool up = tile < T0;
        nup += up;
        const int tt = up ? tile : tile - T0;
        const int tm = up ? tt / tn0 : tt / tn1, tn = up ? tt % tn0 : tt % tn1;
        const int m0 = tm * 256 + rank * 128, n0 = tn * kPairBN + rank * 128;
        const CUtensorMap* ma = up ? &map_a0 : &map_a1;
        const CUtensorMap* mb = up ? &map_b0 : &map_b1;
        if (!up && m0 < M) {   // this unit's lin1 outputs published (all tn0 tiles)
          const long long w0 = f.prof ? clock64() : 0;
          dep_wait_geq(f.ready + tm * 2 + rank, tn0);
          fence_proxy_async_global();
          if (f.prof) wdep += clock64() - w0;
        }
        const int nkb = up ? kb0 : kb1;
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait_sleep(&empty[s], ph ^ 1);
          uint8_t* sa = smem + s * Cf::STAGE_BYTES;
          if (rank == 0) mbar_expect_tx(&full[s], 2 * Cf::STAGE_BYTES);
          const uint32_t fb = mapa_shared(smem_u32(&full[s]), 0);
          tma_load_2d_pair(sa, ma, fb, kb * kBK, m0);
          tma_load_2d_pair(sa + Cf::A_BYTES, mb, fb, kb * kBK, n0);
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
      }
      if (f.prof && rank == 0) {
        f.prof[(blockIdx.x >> 1) * 8 + 4] = wdep;
        f.prof[(blockIdx.x >> 1) * 8 + 5] = nup;
      }
    }
  } else if (warp == 1) {
    // ===== MMA issuer (leader)
    if (rank == 0) {
      constexpr uint32_t idesc = idesc_bf16_f32(256, kPairBN);
      int s = 0, t = 0;
      uint32_t ph = 0;
      const uint64_t a_desc0 = sdesc_k_sw128(smem_u32(smem));
      long long w_acc = 0, w_full = 0, mma_ideal = 0;
      const long long t0c = clock64();
      for (;; ++t) {
        int tile = 0;
        if (lane == 0) tile = read_tile(t, true);
        tile = __shfl_sync(0xffffffffu, tile, 0);
        if (tile >= num_tiles) break;
        const int nkb = tile < T0 ? kb0 : kb1;
        mma_ideal += nkb * 512;
        const int acc = t & 1;
        {
          const long long a = clock64();
          mbar_wait(&acc_empty[acc], ((t >> 1) & 1) ^ 1);
          w_acc += clock64() - a;
        }
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * kPairBN;
        for (int kb = 0; kb < nkb; ++kb) {
          {
            const long long a = clock64();
            mbar_wait(&full[s], ph);
            w_full += clock64() - a;
          }
          tc_fence_after();
          const uint64_t ad = a_desc0 + (uint64_t)s * (uint64_t)(Cf::STAGE_BYTES >> 4);
          const uint64_t bd = ad + (uint64_t)(Cf::A_BYTES >> 4);
          if (elect_one_sync()) {
#pragma unroll
            for (int kk = 0; kk < kBK / 16; ++kk)
              umma_bf16_pair(d_tmem, ad + (uint64_t)(kk * 2), bd + (uint64_t)(kk * 2), idesc, (kb | kk) != 0);
            umma_commit_pair(&empty[s], 3);
          }
          __syncwarp();
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
        if (elect_one_sync()) umma_commit_pair(&acc_full[acc], 3);
        __syncwarp();
      }
      if (f.prof && lane == 0) {
        long long* pp = f.prof + (blockIdx.x >> 1) * 8;
        pp[0] = clock64() - t0c;
        pp[1] = w_acc;
        pp[2] = w_full;
        pp[3] = t;
        pp[6] = mma_ideal;
      }
    }
  } else if (warp == 2 + EW) {
    // ===== tile scheduler (leader): claims in row-block order, one tile ahead
    if (rank == 0 && lane == 0) {
      const uint32_t peer_full0 = mapa_shared(smem_u32(&tile_full[0]), 1);
      const uint32_t peer_ring0 = mapa_shared(smem_u32(&tile_ring[0]), 1);
      for (int i = 0;; ++i) {
        const int slot = i & 3;
        if (i > 0) mbar_wait(&tile_took[(i - 1) & 3], ((i - 1) >> 2) & 1);
        mbar_wait(&tile_empty[slot], ((i >> 2) & 1) ^ 1);
        const int tile = atomicAdd(f.tiles, 1);
        tile_ring[slot] = tile;
        st_shared_cluster_s32(peer_ring0 + slot * 4, tile);
        mbar_arrive(&tile_full[slot]);
        mbar_arrive_cluster(peer_full0 + slot * 8);
        if (tile >= num_tiles) break;
      }
    }
  } else {
    // ===== epilogue warps (both CTAs): lin1 = LayerNorm correction + bias + GELU,
    // lin2 = bias + LayerNorm'd residual + output statistics; SW64 boxes, TMA stores
    const int quarter = warp & 3;
    const int part = (warp - 2) >> 2;
    const int ew = warp - 2;
    const uint32_t leader_empty0 = mapa_shared(smem_u32(&acc_empty[0]), 0);
    for (int i = threadIdx.x - 64; i < f.n_up; i += 32 * EW) {
      bias0_s[i] = __ldg(f.bias0 + i);
      aux0_s[i] = __ldg(f.colsum0 + i);
    }
    for (int i = threadIdx.x - 64; i < f.n_down; i += 32 * EW) {
      bias1_s[i] = __ldg(f.bias1 + i);
      aux1_s[i] = __ldg(f.r_gamma + i);
      aux1_s[f.n_down + i] = __ldg(f.r_beta + i);
    }
    asm volatile("bar.sync 1, %0;" ::"n"(32 * EW) : "memory");
    uint8_t* stg = stg_base + ew * (2 * 2048);
    uint64_t* rb = res_full + ew * 2;
    uint32_t rph = 0;
    const int sw = (lane >> 1) & 3;
    int pending = -1;   // unit of a lin1 tile whose stores may still be in flight
    int tile = 0;
    if (lane == 0) tile = read_tile(0, true);
    tile = __shfl_sync(0xffffffffu, tile, 0);
    for (int t = 0; tile < num_tiles; ++t) {
      const bool up = tile < T0;
      const int tt = up ? tile : tile - T0;
      const int tm = up ? tt / tn0 : tt / tn1, tn = up ? tt % tn0 : tt % tn1;
      const int acc = t & 1;
      const int row0 = tm * 256 + rank * 128 + quarter * 32;
      const int colw = tn * kPairBN + part * CW;
      const bool rows_ok = row0 < M;
      if (!up && rows_ok && lane == 0) {   // residual of chunk 0
        bulk_wait_read<0>();
        mbar_expect_tx(&rb[0], 2048);
        tma_load_2d(stg, &map_r1, &rb[0], colw, row0);
      }
      float a_sc = 1.0f, a_sh = 0.0f;   // lin1: LN of the input rows; lin2: LN of the residual rows
      if (rows_ok)
        ln_row_params(up ? f.a_stats : f.r_stats, f.parts, f.ln_ld, row0 + lane, f.n_down, f.eps, a_sc, a_sh);
      float st_k = 0.0f, st_s1 = 0.0f, st_s2 = 0.0f;
      int ngroups = 0;
      mbar_wait_sleep(&acc_full[acc], (t >> 1) & 1);
      tc_fence_after();
      const uint32_t tacc = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * kPairBN + part * CW;
#pragma unroll 1
      for (int c = 0; c < NCH; ++c) {
        const int b = c & 1;
        uint8_t* buf = stg + b * 2048;
        if (!up && rows_ok && lane == 0 && c + 1 < NCH) {
          bulk_wait_read<0>();
          mbar_expect_tx(&rb[b ^ 1], 2048);
          tma_load_2d(stg + (b ^ 1) * 2048, &map_r1, &rb[b ^ 1], colw + 32 * (c + 1), row0);
        }
        uint32_t r[32];
        tmem_ld_32x32b_x32(tacc + 32 * c, r);
        tmem_ld_wait();
        if (!rows_ok) continue;
        const int col0 = colw + 32 * c;
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
        uint4* myrow = reinterpret_cast<uint4*>(buf + lane * 64);
        if (up) {
          const uint64_t sc2 = f2_pack(a_sc, a_sc), sh2 = f2_pack(a_sh, a_sh);
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            const float4 sj = *reinterpret_cast<const float4*>(aux0_s + col0 + i);
            const float4 cj = *reinterpret_cast<const float4*>(bias0_s + col0 + i);
            const uint64_t t0 = f2_fma(sh2, f2_pack(sj.x, sj.y), f2_pack(cj.x, cj.y));
            const uint64_t t1 = f2_fma(sh2, f2_pack(sj.z, sj.w), f2_pack(cj.z, cj.w));
            f2_unpack(f2_fma(sc2, f2_pack(v[i], v[i + 1]), t0), v[i], v[i + 1]);
            f2_unpack(f2_fma(sc2, f2_pack(v[i + 2], v[i + 3]), t1), v[i + 2], v[i + 3]);
          }
#pragma unroll
          for (int i = 0; i < 32; i += 2) gelu_erf2(v[i], v[i + 1]);
          // the store that last read this buffer (two chunks ago) is done
          if (lane == 0) bulk_wait_read<1>();
          __syncwarp();
        } else {
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            const float4 bb = *reinterpret_cast<const float4*>(bias1_s + col0 + i);
            f2_unpack(f2_add(f2_pack(v[i], v[i + 1]), f2_pack(bb.x, bb.y)), v[i], v[i + 1]);
            f2_unpack(f2_add(f2_pack(v[i + 2], v[i + 3]), f2_pack(bb.z, bb.w)), v[i + 2], v[i + 3]);
          }
          mbar_wait(&rb[b], (rph >> b) & 1u);
          rph ^= 1u << b;
          const uint64_t sc2 = f2_pack(a_sc, a_sc), sh2 = f2_pack(a_sh, a_sh);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint4 u = myrow[q ^ sw];
            const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&u);
            const int cc = col0 + q * 8;
            const float4 g0 = *reinterpret_cast<const float4*>(aux1_s + cc);
            const float4 g1 = *reinterpret_cast<const float4*>(aux1_s + cc + 4);
            const float4 b0 = *reinterpret_cast<const float4*>(aux1_s + f.n_down + cc);
            const float4 b1 = *reinterpret_cast<const float4*>(aux1_s + f.n_down + cc + 4);
            const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
            const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
            for (int e = 0; e < 8; e += 2) {
              const float2 fr = __bfloat1622float2(h2[e >> 1]);
              const uint64_t nrm = f2_fma(f2_pack(fr.x, fr.y), sc2, sh2);
              const uint64_t rr = f2_fma(nrm, f2_pack(gg[e], gg[e + 1]), f2_pack(bb[e], bb[e + 1]));
              f2_unpack(f2_add(f2_pack(v[q * 8 + e], v[q * 8 + e + 1]), rr), v[q * 8 + e], v[q * 8 + e + 1]);
            }
          }
        }
        uint4 u[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          u[q].x = pack_bf16(v[q * 8 + 0], v[q * 8 + 1]);
          u[q].y = pack_bf16(v[q * 8 + 2], v[q * 8 + 3]);
          u[q].z = pack_bf16(v[q * 8 + 4], v[q * 8 + 5]);
          u[q].w = pack_bf16(v[q * 8 + 6], v[q * 8 + 7]);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) myrow[q ^ sw] = u[q];
        if (!up) {   // lin2 output row statistics (shifted sums of the fp32 values)
          if (c == 0) st_k = v[0];
          const uint64_t nk = f2_pack(-st_k, -st_k);
          uint64_t s1 = f2_pack(0.0f, 0.0f), s2 = f2_pack(0.0f, 0.0f);
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            const uint64_t d = f2_add(f2_pack(v[i], v[i + 1]), nk);
            s1 = f2_add(s1, d);
            s2 = f2_fma(d, d, s2);
          }
          float a0, a1, c0, c1;
          f2_unpack(s1, a0, a1);
          f2_unpack(s2, c0, c1);
          st_s1 += a0 + a1;
          st_s2 += c0 + c1;
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_2d(up ? &map_o0 : &map_o1, buf, col0, row0);
          bulk_commit();
        }
        ++ngroups;
      }
      if (!up && rows_ok) {
        const float n = (float)CW;
        const float mi = st_k + st_s1 / n;
        const float m2 = fmaxf(st_s2 - st_s1 * st_s1 / n, 0.0f);
        f.out_stats[(int64_t)(tn * PARTS + part) * f.ln_ld + row0 + lane] = make_float2(mi, m2);
      }
      tc_fence_before();
      asm volatile("bar.sync 1, %0;" ::"n"(32 * EW) : "memory");
      if (threadIdx.x == 64) {
        if (rank == 0) mbar_arrive(&acc_empty[acc]);
        else mbar_arrive_cluster(leader_empty0 + acc * 8);
      }
      // Publication of lin1 tiles for their units' lin2 tiles, one tile late (the
      // stores had a tile's time to land) -- except before this pair's first lin2
      // tile or the end, which may wait on this very tile: then at once.
      int next = 0;
      if (lane == 0) next = read_tile(t + 1, true);
      next = __shfl_sync(0xffffffffu, next, 0);
      const int unit = tm * 2 + (int)rank;
      const bool valid_unit = tm * 256 + (int)rank * 128 < M;
      const bool flush_now = up && (next >= T0);
      if (pending >= 0 || flush_now) {
        if (lane == 0) {
          if (flush_now || ngroups == 0) bulk_wait<0>();
          else if (ngroups == 1) bulk_wait<1>();
          else if (ngroups == 2) bulk_wait<2>();
          else if (ngroups == 3) bulk_wait<3>();
          else bulk_wait<4>();
          fence_proxy_async_global();
        }
        asm volatile("bar.sync 1, %0;" ::"n"(32 * EW) : "memory");
        if (threadIdx.x == 64) {
          if (pending >= 0) dep_signal_add_nofence(f.ready + pending, 1);
          if (flush_now && valid_unit) dep_signal_add_nofence(f.ready + unit, 1);
        }
      }
      pending = (up && !flush_now && valid_unit) ? unit : -1;
      tile = next;
    }
    if (lane == 0) bulk_wait<0>();
  }
  __syncthreads();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, 2 * kPairBN);
  }
}

template <int STAGES, int EW, int NBUF, int EK>
static int launch_gemm_pair(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mo,
                            const CUtensorMap& mr, int M, int N, int K, const GemmEpilogue& ep,
                            cudaStream_t s) {
  using Cf = PairCfg<STAGES, EW, NBUF, EK>;
  auto kern = gemm_bf16_pair<STAGES, EW, NBUF, EK>;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cf::SMEM) != cudaSuccess)
      return GG_ERR_CUDA;
    attr = true;
  }
  const int tiles = ((M + 255) / 256) * (N / kPairBN);
  const int pairs = num_sms() / 2;
  const int grid = 2 * (tiles < pairs ? tiles : pairs);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(Cf::kThreads);
  cfg.dynamicSmemBytes = Cf::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  static long long* prof = nullptr;
  GemmEpilogue e2 = ep;
  const bool do_prof = getenv("GG_GEMM_PROF") != nullptr;
  if (do_prof) {
    e2.dbg_skip_epi = getenv("GG_GEMM_SKIP_EPI") != nullptr;
    if (!prof) cudaMalloc(&prof, 4096 * sizeof(long long));
    cudaMemsetAsync(prof, 0, 4096 * sizeof(long long), s);
    e2.prof = prof;
  }
  if (cudaLaunchKernelEx(&cfg, kern, ma, mb, mo, mr, M, N, K, e2) != cudaSuccess) return GG_ERR_CUDA;
  GG_LAUNCH_OK();
  if (do_prof) {
    long long h[4096];
    cudaDeviceSynchronize();
    cudaMemcpy(h, prof, sizeof(h), cudaMemcpyDeviceToHost);
    double tot = 0, wa = 0, wf = 0, nt = 0;
    long long e0 = LLONG_MAX, e1 = 0, w1 = 0, i1 = 0, x1 = 0;
    const int np = grid / 2;
    double ghz = 0;
    for (int i = 0; i < np; ++i)
      ghz += (double)(h[2048 + 2 * i + 1] - h[2048 + 2 * i]) / (double)(h[8 * i + 7] - h[8 * i + 4]) / np;
    for (int i = 0; i < np; ++i) {
      tot += h[8 * i];
      wa += h[8 * i + 1];
      wf += h[8 * i + 2];
      nt += h[8 * i + 3];
      e0 = h[8 * i + 4] < e0 ? h[8 * i + 4] : e0;
      e1 = h[8 * i + 4] > e1 ? h[8 * i + 4] : e1;
      w1 = h[8 * i + 5] > w1 ? h[8 * i + 5] : w1;
      i1 = h[8 * i + 6] > i1 ? h[8 * i + 6] : i1;
      x1 = h[8 * i + 7] > x1 ? h[8 * i + 7] : x1;
    }
    fprintf(stderr, "pair GEMM<EW=%d,EK=%d> M=%d N=%d K=%d: issuer %.0f cycles/pair, %.2f tiles/pair, "
            "waiting acc_empty %.0f%%, operands %.0f%%, MMA-bound ideal %.0f cycles; timeline (us from the "
            "first CTA): last CTA in %.2f, prologue done %.2f, last MMA issued %.2f, last epilogue %.2f; SM %.2f GHz%s\n",
            EW, EK, M, N, K, tot / np, nt / np, 100 * wa / tot, 100 * wf / tot,
            nt / np * (K / kBK) * 4 * 128.0, (e1 - e0) * 1e-3, (w1 - e0) * 1e-3, (i1 - e0) * 1e-3,
            (x1 - e0) * 1e-3, ghz, e2.dbg_skip_epi ? " [epilogue skipped]" : "");
  }
  return GG_OK;
}

// Epilogue kind -> instantiation.  Residual kernels keep 8 epilogue warps and
// two staging boxes per warp (the residual box of the next chunk in flight);
// the others run 16 epilogue warps (two chunks each) so the GELU / LayerNorm
// correction math of a tile keeps pace with the next tile's MMAs.
static int g_pair_ew = -1;
static int pair_ew() {
  if (g_pair_ew < 0) g_pair_ew = getenv("GG_PAIR_EW") ? atoi(getenv("GG_PAIR_EW")) : 16;
  return g_pair_ew;
}

template <int EK>
static int launch_pair_kind(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mo,
                            const CUtensorMap& mr, int M, int N, int K, const GemmEpilogue& ep,
                            cudaStream_t s) {
  if constexpr ((EK & EK_RES) != 0) {
    return launch_gemm_pair<5, 8, 2, EK>(ma, mb, mo, mr, M, N, K, ep, s);
  } else {
    if (pair_ew() == 8) return launch_gemm_pair<5, 8, 1, EK>(ma, mb, mo, mr, M, N, K, ep, s);
    if constexpr (EK == (EK_ALN | EK_GELU) || EK == (EK_QKV | EK_ALN)) {
      // QKV and FFN-up with LayerNorm folding (K = 768): 4 operand stages and two
      // staging boxes per epilogue warp (a warp's next chunk no longer waits for its
      // previous TMA store to drain the box): QKV 47.3 -> 45.6 us, FFN-up 64.1 -> 63.7
      // (no-PDL CUPTI); the layer-0 QKV (no folding) measured slower this way
      static const bool nb1 = getenv("GG_PAIR_NB1") != nullptr;   // the 5-stage, one-box form
      if (!nb1) return launch_gemm_pair<4, 16, 2, EK>(ma, mb, mo, mr, M, N, K, ep, s);
    }
    return launch_gemm_pair<5, 16, 1, EK>(ma, mb, mo, mr, M, N, K, ep, s);
  }
}

static int launch_pair(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mo,
                       const CUtensorMap& mr, int M, int N, int K, const GemmEpilogue& ep, cudaStream_t s) {
  const int ek = (ep.a_stats ? EK_ALN : 0) | (ep.act == ACT_GELU ? EK_GELU : 0) |
                 (ep.residual ? EK_RES : 0) | (ep.out_mode == OUT_QKV_HEADS ? EK_QKV : 0);
  switch (ek) {
#define GG_PAIR_CASE(k) \
  case k: return launch_pair_kind<k>(ma, mb, mo, mr, M, N, K, ep, s);
    GG_PAIR_CASE(0) GG_PAIR_CASE(1) GG_PAIR_CASE(2) GG_PAIR_CASE(3) GG_PAIR_CASE(4) GG_PAIR_CASE(5)
    GG_PAIR_CASE(6) GG_PAIR_CASE(7) GG_PAIR_CASE(8) GG_PAIR_CASE(9) GG_PAIR_CASE(10) GG_PAIR_CASE(11)
    GG_PAIR_CASE(12) GG_PAIR_CASE(13) GG_PAIR_CASE(14) GG_PAIR_CASE(15)
#undef GG_PAIR_CASE
    default: return GG_ERR_INVALID_ARGUMENT;
  }
}
}  // namespace gg

using namespace gg;

static int gemm_impl(const void* A, int64_t lda, const void* B, int64_t ldb, void* D, int64_t ldd,
                     int64_t M, int64_t N, int64_t K, const gg_gemm_epilogue* e,
                     const gg_gemm_ln_params* ln, const gg_dep* dep, void* stream) {
  if (!A || !B || !D || !e || M <= 0 || N <= 0 || K <= 0) return GG_ERR_INVALID_ARGUMENT;
  if (K % 64 || N % 32 || lda % 8 || ldb % 8 || (e->residual && e->ldr % 8)) return GG_ERR_INVALID_ARGUMENT;
  if (e->act < 0 || e->act > 2 || e->out_mode < 0 || e->out_mode > 2) return GG_ERR_INVALID_ARGUMENT;
  if (e->out_mode == OUT_BF16 && ldd % 8) return GG_ERR_INVALID_ARGUMENT;
  if (e->out_mode == OUT_F32 && ldd % 4) return GG_ERR_INVALID_ARGUMENT;
  if (e->out_mode == OUT_QKV_HEADS &&
      (e->seq_len <= 0 || e->heads <= 0 || N != 3 * 64 * (int64_t)e->heads || M % e->seq_len ||
       e->seq_len % 128))
    return GG_ERR_INVALID_ARGUMENT;
  int bn = e->tile_n > 0 ? e->tile_n : (N % 256 == 0 ? 256 : (N % 128 == 0 ? 128 : 64));
  if (bn != 64 && bn != 128 && bn != 256) return GG_ERR_INVALID_ARGUMENT;
  CUtensorMap ma, mb;
  int rc = make_map_2d(&ma, A, M, K, lda, 128);
  if (rc) return rc;
  rc = make_map_2d(&mb, B, N, K, ldb, bn);
  if (rc) return rc;
  if (e->count_dev && e->rows_per_item <= 0) return GG_ERR_INVALID_ARGUMENT;
  GemmEpilogue ep{D, ldd, e->bias, reinterpret_cast<const __nv_bfloat16*>(e->residual), e->ldr,
                  e->act, e->out_mode, e->seq_len, e->heads,
                  e->out_mode == OUT_QKV_HEADS ? M * 64 * (int64_t)e->heads : 0,
                  e->count_dev, e->rows_per_item, StreamK{nullptr, nullptr, 0},
                  M * K * 2 > (48LL << 20) ? 1 : 0, nullptr, 0};
  if (ln) {
    if (ln->ln_width <= 0 || ln->ln_width % 128 || ln->ln_width > kPairAuxFloats / 2)
      return GG_ERR_INVALID_ARGUMENT;
    if ((ln->a_stats && !ln->a_colsum) || (ln->r_stats && (!ln->r_gamma || !ln->r_beta || !e->residual)))
      return GG_ERR_INVALID_ARGUMENT;
    if (ln->a_stats && (ln->ln_width != K || N > kPairAuxFloats)) return GG_ERR_INVALID_ARGUMENT;
    if ((ln->r_stats || ln->out_stats) && ln->ln_width != N) return GG_ERR_INVALID_ARGUMENT;
    if (ln->out_stats && !e->residual) return GG_ERR_UNSUPPORTED;   // statistics ride the residual epilogue
    ep.a_stats = reinterpret_cast<const float2*>(ln->a_stats);
    ep.a_colsum = ln->a_colsum;
    ep.r_stats = reinterpret_cast<const float2*>(ln->r_stats);
    ep.r_gamma = ln->r_gamma;
    ep.r_beta = ln->r_beta;
    ep.out_stats = reinterpret_cast<float2*>(ln->out_stats);
    ep.a_parts = ep.r_parts = ln->ln_width / 128;
    ep.ln_width = ln->ln_width;
    ep.ln_ld = M;
    ep.eps = ln->eps;
  }
  if (dep && (dep->wait || dep->signal)) {
    // tile-level dependencies live in the CTA-pair kernel; units of 128 rows
    if (M % 128 || (e->count_dev && e->rows_per_item % 128) || (dep->wait && dep->need <= 0) || !dep->go)
      return GG_ERR_INVALID_ARGUMENT;
    ep.dep_wait = dep->wait;
    ep.dep_need = dep->need;
    ep.dep_signal = dep->signal;
    ep.dep_go = dep->go;
    ep.dep_tiles = dep->tiles;
    static const int dbg = getenv("GG_DEP_DBG") ? atoi(getenv("GG_DEP_DBG")) : 0;
    ep.dep_dbg = dbg;
    ep.raster_n = 1;   // row blocks in order: the consumer's readiness follows the producer's
  }
  const bool want_dep = ep.dep_wait || ep.dep_signal;
  static const int raster_env = getenv("GG_RASTER_N") ? atoi(getenv("GG_RASTER_N")) : -1;
  if (raster_env >= 0) ep.raster_n = raster_env;
  cudaStream_t s = gg_stream(stream);
  // CTA pairs for wide GEMMs (tile_n auto, N % 256 == 0, enough 256-row tiles
  // to fill most pairs); GG_NO_PAIR=1 keeps single-CTA tiles
  static const bool no_pair = getenv("GG_NO_PAIR") != nullptr;
  if (!no_pair && e->tile_n == 0 && N % kPairBN == 0 && N <= kPairMaxN && M >= 256 * 16) {
    CUtensorMap mbp, mo, mr;
    rc = make_map_2d(&ma, A, M, K, lda, 128);
    if (!rc) rc = make_map_2d(&mbp, B, N, K, ldb, 128);
    if (rc) return rc;
    // outputs / residuals through smem + TMA (bf16 outputs; dynamic row counts in
    // multiples of 32 so a 32-row box is all valid or all beyond the batch)
    static const bool no_tma_out = getenv("GG_NO_TMA_EPI") != nullptr;
    const bool tma_ok = !no_tma_out && (e->out_mode == OUT_BF16 || e->out_mode == OUT_QKV_HEADS) &&
                        (!e->count_dev || e->rows_per_item % 32 == 0);
    if (tma_ok) {
      mr = ma;
      if (e->out_mode == OUT_BF16) rc = make_map_box32(&mo, D, M, N, ldd);
      else {   // Q / K planes as [3 B H S, 64]; the V^T plane [B H 64, S] in the residual slot
        rc = make_map_box32(&mo, D, 3 * M * (int64_t)e->heads, 64, 64);
        if (!rc)
          rc = make_map_box32(&mr, reinterpret_cast<__nv_bfloat16*>(D) + 2 * M * 64 * (int64_t)e->heads,
                              M / e->seq_len * e->heads * 64, e->seq_len, e->seq_len);
      }
      if (!rc && e->residual) rc = make_map_box32(&mr, e->residual, M, N, e->ldr);
      if (rc) return rc;
      ep.tma_out = 1;
      return launch_pair(ma, mbp, mo, mr, (int)M, (int)N, (int)K, ep, s);
    }
    if (want_dep) return GG_ERR_UNSUPPORTED;
    // (no TMA epilogue: the single-CTA kernel below)
    rc = make_map_2d(&ma, A, M, K, lda, 128);
    if (rc) return rc;
  }
  if (ln || want_dep) return GG_ERR_UNSUPPORTED;   // LayerNorm folding / deps live in the CTA-pair kernel
  switch (bn) {
    case 256: return launch_gemm<128, 256, 4>(ma, mb, (int)M, (int)N, (int)K, ep, s, 0);
    case 128: return launch_gemm<128, 128, 6>(ma, mb, (int)M, (int)N, (int)K, ep, s, 0);
    default: return launch_gemm<128, 64, 8>(ma, mb, (int)M, (int)N, (int)K, ep, s, 0);
  }
}

extern "C" int gg_gemm(const void* A, int64_t lda, const void* B, int64_t ldb, void* D,
                       int64_t ldd, int64_t M, int64_t N, int64_t K, const gg_gemm_epilogue* e,
                       void* stream) {
  return gemm_impl(A, lda, B, ldb, D, ldd, M, N, K, e, nullptr, nullptr, stream);
}

extern "C" int gg_gemm_ln(const void* A, int64_t lda, const void* B, int64_t ldb, void* D,
                          int64_t ldd, int64_t M, int64_t N, int64_t K, const gg_gemm_epilogue* e,
                          const gg_gemm_ln_params* ln, void* stream) {
  if (!ln) return GG_ERR_INVALID_ARGUMENT;
  return gemm_impl(A, lda, B, ldb, D, ldd, M, N, K, e, ln, nullptr, stream);
}

extern "C" int gg_gemm_dep(const void* A, int64_t lda, const void* B, int64_t ldb, void* D,
                           int64_t ldd, int64_t M, int64_t N, int64_t K, const gg_gemm_epilogue* e,
                           const gg_gemm_ln_params* ln, const gg_dep* dep, void* stream) {
  if (!dep) return GG_ERR_INVALID_ARGUMENT;
  return gemm_impl(A, lda, B, ldb, D, ldd, M, N, K, e, ln, dep, stream);
}


extern "C" int gg_ffn_pair(const void* A, const void* W1, void* H, const void* W2, void* Y,
                           int64_t M, int32_t d, int32_t F, const int32_t* count_dev,
                           int32_t rows_per_item, const float* bias1, const float* colsum1,
                           const float* a_stats, const float* bias2, const float* r_stats,
                           const float* ln_gamma, const float* ln_beta, float* out_stats, float eps,
                           int32_t* ready, int32_t* tiles, void* stream) {
  if (!A || !W1 || !H || !W2 || !Y || !bias1 || !colsum1 || !a_stats || !bias2 || !r_stats ||
      !ln_gamma || !ln_beta || !out_stats || !ready || !tiles || M <= 0)
    return GG_ERR_INVALID_ARGUMENT;
  if (d % kPairBN || F % kPairBN || d > kFfnMaxDown || F > kFfnMaxUp || d % 128 || M % 128 ||
      M > 0x7fffffff || (count_dev && rows_per_item % 128))
    return GG_ERR_UNSUPPORTED;
  CUtensorMap ma0, mb0, mo0, ma1, mb1, mo1, mr1;
  int rc = make_map_2d(&ma0, A, M, d, d, 128);
  if (!rc) rc = make_map_2d(&mb0, W1, F, d, d, 128);
  if (!rc) rc = make_map_box32(&mo0, H, M, F, F);
  if (!rc) rc = make_map_2d(&ma1, H, M, F, F, 128);
  if (!rc) rc = make_map_2d(&mb1, W2, d, F, F, 128);
  if (!rc) rc = make_map_box32(&mo1, Y, M, d, d);
  if (!rc) rc = make_map_box32(&mr1, A, M, d, d);
  if (rc) return rc;
  FfnArgs f;
  f.M_max = (int)M;
  f.count = count_dev;
  f.rows_per_item = count_dev ? rows_per_item : 1;
  f.n_up = F;
  f.n_down = d;
  f.k_up = d;
  f.bias0 = bias1;
  f.colsum0 = colsum1;
  f.a_stats = reinterpret_cast<const float2*>(a_stats);
  f.bias1 = bias2;
  f.r_stats = reinterpret_cast<const float2*>(r_stats);
  f.r_gamma = ln_gamma;
  f.r_beta = ln_beta;
  f.out_stats = reinterpret_cast<float2*>(out_stats);
  f.parts = d / 128;
  f.ln_ld = M;
  f.eps = eps;
  f.ready = ready;
  f.tiles = tiles;
  static long long* prof = nullptr;
  const bool do_prof = getenv("GG_GEMM_PROF") != nullptr;
  f.prof = nullptr;
  if (do_prof) {
    if (!prof) cudaMalloc(&prof, 1024 * sizeof(long long));
    cudaMemsetAsync(prof, 0, 1024 * sizeof(long long), gg_stream(stream));
    f.prof = prof;
  }
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(gemm_ffn_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, FfnCfg::SMEM) !=
        cudaSuccess)
      return GG_ERR_CUDA;
    attr = true;
  }
  const int pairs = num_sms() / 2;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(kFfnThreads);
  cfg.dynamicSmemBytes = FfnCfg::SMEM;
  cfg.stream = gg_stream(stream);
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  if (cudaLaunchKernelEx(&cfg, gemm_ffn_pair, ma0, mb0, mo0, ma1, mb1, mo1, mr1, f) != cudaSuccess)
    return GG_ERR_CUDA;
  GG_LAUNCH_OK();
  if (do_prof) {
    long long h[1024];
    cudaDeviceSynchronize();
    cudaMemcpy(h, prof, sizeof(h), cudaMemcpyDeviceToHost);
    double tot = 0, wa = 0, wf = 0, nt = 0, wd = 0, nu = 0, ideal = 0, tmax = 0, imax = 0;
    for (int i = 0; i < pairs; ++i) {
      tot += h[8 * i]; wa += h[8 * i + 1]; wf += h[8 * i + 2]; nt += h[8 * i + 3];
      wd += h[8 * i + 4]; nu += h[8 * i + 5]; ideal += h[8 * i + 6];
      tmax = h[8 * i] > tmax ? h[8 * i] : tmax;
      imax = h[8 * i + 6] > imax ? h[8 * i + 6] : imax;
    }
    fprintf(stderr, "ffn pair M=%lld: issuer %.0f cycles/pair (max %.0f), MMA-bound %.0f (max %.0f), tiles %.2f/pair "
            "(lin1 %.2f), waiting acc %.0f%% operands %.0f%%, lin2 dependency wait %.0f cycles/pair\n",
            (long long)M, tot / pairs, tmax, ideal / pairs, imax, nt / pairs, nu / pairs, 100 * wa / tot,
            100 * wf / tot, wd / pairs);
  }
  return GG_OK;
}

extern "C" int gg_zero_async(void* ptr, int64_t bytes, void* stream) {
  if (!ptr || bytes < 0) return GG_ERR_INVALID_ARGUMENT;
  return cudaMemsetAsync(ptr, 0, (size_t)bytes, gg_stream(stream)) == cudaSuccess ? GG_OK : GG_ERR_CUDA;
}

extern "C" int gg_streamk_reserve(void) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return GG_ERR_CUDA;
  return sk_alloc(dev) ? GG_OK : GG_ERR_CUDA;
}

extern "C" int gg_streamk_mode(int32_t mode) {
  const int prev = sk_mode();
  if (mode >= -1 && mode <= 1) g_sk_mode = mode;
  return prev;
}

extern "C" int gg_gemm_bf16(const void* A, int64_t lda, const void* B, int64_t ldb, void* D,
                            int64_t ldd, int64_t M, int64_t N, int64_t K, const float* bias,
                            const void* residual, int64_t ldr, int32_t act, int32_t tile_n,
                            void* stream) {
  gg_gemm_epilogue e{bias, residual, ldr, act, OUT_BF16, 0, 0, tile_n, 0, nullptr};
  return gg_gemm(A, lda, B, ldb, D, ldd, M, N, K, &e, stream);
}

// Persistent grids (GEMMs, attention, span convolutions) size themselves to the
// SM count minus `n` (even: CTA pairs) for launches issued -- or captured into a
// graph -- after this call: the pipelined serving loop keeps a TPC free for the
// control stream that runs beside the forward.  Returns the previous value.
extern "C" int gg_set_sm_reserve(int32_t n) {
  const int prev = g_sm_reserve;
  if (n < 0 || (n & 1) || n >= device_sms()) return -1;
  g_sm_reserve = n;
  return prev;
}
