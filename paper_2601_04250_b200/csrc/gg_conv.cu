// gg_conv.cu — ResNet-18 building blocks on sm_100a (NHWC bf16).
//
// Implicit-GEMM convolution on tcgen05:
//   D[m, co] = relu?( sum_k A[m, k] * W[co, k] + bias[co] (+ residual[m, co]) )
//   m = (n, ho, wo) output pixel, k = (r, s, c) with c fastest, W = BN-folded
//   weights [Cout, Kpad] (K-major, zero padded to a multiple of 64).
// The A operand is never materialized: producer warps gather each 128-pixel x
// 64-k tile straight from the NHWC activation with 16-byte cp.async (zero-fill
// for padding and K tail) into the 128B-swizzled layout tcgen05 reads; B comes
// in by TMA; the fp32 accumulator lives in TMEM (double buffered, persistent
// CTAs); the epilogue fuses folded-BN bias, the residual add and ReLU.
//
//   warps 0-3  A gather (cp.async) + warp 0 lane 0 B TMA
//   warp 4     TMEM allocator + MMA issuer
//   warps 5-8  epilogue
#include <cudaTypedefs.h>

#include "gg_common.cuh"
#include "gg_kernels.h"
#include "gg_streamk.cuh"
#include "gg_tc.cuh"
#include "gg_act.cuh"

namespace gg {
using namespace tc;

struct ConvShape {
  int N, H, W, C;      // input NHWC (C multiple of 8)
  int Ho, Wo, Cout;
  int R, S, stride, pad;
  int pad_hi;          // bottom/right padding (== pad for symmetric convolutions)
  int bres;            // resident-B mode (weights loaded once per CTA)
  int bres_stages;     // A-ring depth in resident-B mode
  int Kpad;            // multiple of 64, >= R*S*C
  int M;               // N*Ho*Wo
};

struct ConvEpi {
  act_t* y;               // [M, Cout]
  const float* bias;              // [Cout]
  const act_t* residual;  // [M, Cout] or null
  int relu;
  const int32_t* count;           // device image count (dynamic batch) or null
  int out_pad;                    // 1: y (and residual) are [N, Ho+2, Wo+2, Cout] zero-bordered
  StreamK sk;                     // stream-K split (TMA im2col mode only), or disabled
  act_t* y_ds;            // DS: the fused 1x1 / stride-2 downsample output (no ReLU)
  const float* bias_ds;           // DS: its folded-BN bias
};

constexpr int kConvProdWarps = 4;
// epilogue warps: 4 (one per TMEM lane quarter); the fused conv + downsample has
// twice the accumulator columns per tile and uses 8 (two column halves)
constexpr int kConvThreadsMax = 32 * (kConvProdWarps + 1 + 8);
__host__ __device__ constexpr int conv_epi_warps(bool ds) { return ds ? 8 : 4; }
constexpr int kLag = 2;  // cp.async groups in flight per producer thread

template <int BN, int STAGES, bool DS = false>
struct ConvSmem {
  static constexpr int A_BYTES = 128 * 128;
  static constexpr int B_BYTES = BN * 128;
  // DS: a second weight slab per stage (the downsample's, used at the centre tap)
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  // DS: the downsample's weight slabs (used by the centre-tap k-blocks only) have
  // their own 2-slot ring after the stages, so every stage stays A + B
  static constexpr int DS_SLOTS = DS ? 2 : 0;
  static constexpr int BAR_OFF = STAGES * STAGE_BYTES + DS_SLOTS * B_BYTES;
  static constexpr int TOTAL = BAR_OFF + 256 + 1024;
};

__device__ __forceinline__ void cp_async_16(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
               "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// MODE 0: cp.async gather (any C % 8 == 0).
// MODE 1 (C % 64 == 0): the A tile of tap (r, s) and channel block c0 is ONE
//   TMA im2col load (cp.async.bulk.tensor.4d...im2col): 128 consecutive output
//   pixels (row/image wrap and zero padding done by the TMA unit) x 64
//   channels, 128B-swizzled.
// MODE 2 (C == 16, the space-to-depth stem): a 64-wide k-block is 4 taps; each
//   tap is one im2col load of 128 pixels x 16 channels (32B-swizzled) that one
//   UMMA K-step consumes.
// DS (MODE 1, 3x3 / stride 2 on a padded input): the block's 1x1 / stride-2
//   downsample reads exactly the centre tap's A tiles, so it rides along — a
//   second weight slab per centre-tap stage and a second TMEM accumulator — instead
//   of a separate kernel re-loading the input.
template <int BN, int STAGES, int MODE, bool DS = false>
__global__ void __launch_bounds__(kConvThreadsMax, 1)
    conv_bf16_tcgen05(const act_t* __restrict__ x, const __grid_constant__ CUtensorMap map_w,
                      const __grid_constant__ CUtensorMap map_x, const __grid_constant__ CUtensorMap map_wds,
                      ConvShape sh, ConvEpi ep) {
  static_assert(!DS || (MODE == 1 && 4 * BN <= 512), "DS: TMA im2col, two double-buffered accumulators");
  using L = ConvSmem<BN, STAGES, DS>;
  constexpr int NACC_COLS = (DS ? 2 : 1) * BN;   // TMEM columns per accumulator buffer
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_align1k(smem_raw);
  // Resident-B mode (sh.bres, im2col modes, one N tile): the whole BN x Kpad
  // weight slab is loaded once per CTA after a shorter A ring and never re-read
  // from L2; the ring then carries only A tiles.
  const int num_kb = sh.Kpad / 64;
  const int nst = sh.bres ? sh.bres_stages : STAGES;
  uint8_t* bres = smem + nst * L::STAGE_BYTES;
  uint8_t* ds_ring = smem + STAGES * L::STAGE_BYTES;   // DS weight slots (never with bres)
  const int bar_off = sh.bres ? nst * L::STAGE_BYTES + num_kb * L::B_BYTES : L::BAR_OFF;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + bar_off);
  uint64_t* empty = full + STAGES;
  uint64_t* acc_full = empty + STAGES;
  uint64_t* acc_empty = acc_full + 2;
  uint64_t* b_full = acc_empty + 2;
  uint64_t* ds_full = b_full + 1;
  uint64_t* ds_empty = ds_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ds_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  griddep_launch();   // the successor may begin its prologue as SMs free up
  const int tiles_n = sh.Cout / BN;
  const bool b_loaded = MODE != 0 && sh.bres &&
                        (ep.sk.enabled || (sh.M + 127) / 128 * tiles_n > (int)blockIdx.x);

  if (threadIdx.x == 0) {
    mbar_init(b_full, 1);
    for (int s = 0; s < STAGES; ++s) {
      // gather mode: 128 producer arrivals + the B TMA arrive; im2col mode: one expect_tx arrive
      mbar_init(&full[s], MODE != 0 ? 1 : 32 * kConvProdWarps + 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&acc_full[a], 1);
      mbar_init(&acc_empty[a], conv_epi_warps(DS));
      mbar_init(&ds_full[a], 1);
      mbar_init(&ds_empty[a], 1);
    }
    fence_mbar_init();
    tma_prefetch(&map_w);
  }
  if (warp == kConvProdWarps) tmem_alloc(tmem_slot, 2 * NACC_COLS);
  if (b_loaded && threadIdx.x == 0) {   // weights: independent of the predecessor
    mbar_expect_tx(b_full, num_kb * L::B_BYTES);
    for (int kb = 0; kb < num_kb; ++kb) tma_load_2d(bres + kb * L::B_BYTES, &map_w, b_full, kb * 64, 0);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  griddep_wait();   // activations, residual, count and output follow the predecessor
  const int M = ep.count ? min(sh.M, __ldg(ep.count) * sh.Ho * sh.Wo) : sh.M;
  const int tiles_m = (M + 127) / 128;
  const int num_tiles = tiles_m * tiles_n;

  if (MODE != 0 && warp < kConvProdWarps) {
    // ===== TMA producer (im2col A + tiled B) =====
    if (threadIdx.x == 0) {
      tma_prefetch(&map_x);
      // lean like the issuer: stage / phase and (tap, channel block) advance incrementally
      const int cblocks = sh.C / 64;
      const int ctap = (sh.R * sh.S) / 2;
      int s = 0, dsl = 0;
      uint32_t ph = 0, dph = 0;
      SkSched sc(ep.sk.enabled, num_tiles, num_kb, blockIdx.x, gridDim.x);
      SkWork w;
      while (sc.next(w)) {
        const int tm = w.tile % tiles_m, tn = w.tile / tiles_m;
        const int m0 = tm * 128;
        const int n0 = m0 / (sh.Ho * sh.Wo);
        const int rem = m0 - n0 * sh.Ho * sh.Wo;
        const int ho0 = rem / sh.Wo, wo0 = rem - (rem / sh.Wo) * sh.Wo;
        const int wc = wo0 * sh.stride - sh.pad, hc = ho0 * sh.stride - sh.pad;
        // MODE 1: k-block kb = (tap, channel block cb); MODE 2: taps 4 kb .. 4 kb + 3
        int tap = MODE == 1 ? w.kb0 / cblocks : w.kb0 * 4;
        int cb = MODE == 1 ? w.kb0 - tap * cblocks : 0;
        int rr = tap / sh.S, ss = tap - rr * sh.S;
        for (int kb = w.kb0; kb < w.kb1; ++kb) {
          mbar_wait_sleep(&empty[s], ph ^ 1);
          uint8_t* sa = smem + s * L::STAGE_BYTES;
          {
            const uint32_t bytes = sh.bres ? L::A_BYTES : L::A_BYTES + L::B_BYTES;
            mbar_expect_tx(&full[s], bytes);
          }
          constexpr int kLoads = MODE == 1 ? 1 : 4;
#pragma unroll
          for (int q = 0; q < kLoads; ++q) {
            asm volatile(
                "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};" ::"r"(smem_u32(sa + q * 4096)),
                "l"(&map_x), "r"(smem_u32(&full[s])), "r"(cb * 64), "r"(wc), "r"(hc), "r"(n0),
                "h"((uint16_t)ss), "h"((uint16_t)rr)
                : "memory");
            if (MODE == 2) {   // next tap
              if (++ss == sh.S) {
                ss = 0;
                ++rr;
              }
            }
          }
          if (!sh.bres) tma_load_2d(sa + L::A_BYTES, &map_w, &full[s], kb * 64, tn * BN);
          if constexpr (DS) {   // centre tap: the downsample's weights for this channel block
            if (tap == ctap) {
              mbar_wait_sleep(&ds_empty[dsl], dph ^ 1);
              mbar_expect_tx(&ds_full[dsl], L::B_BYTES);
              tma_load_2d(ds_ring + dsl * L::B_BYTES, &map_wds, &ds_full[dsl], cb * 64, tn * BN);
              if (++dsl == 2) {
                dsl = 0;
                dph ^= 1;
              }
            }
          }
          if (MODE == 1 && ++cb == cblocks) {   // next (tap, channel block)
            cb = 0;
            ++tap;
            if (++ss == sh.S) {
              ss = 0;
              ++rr;
            }
          }
          if (MODE == 2) tap += 4;
          if (++s == nst) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp < kConvProdWarps) {
    // ===== A gather: thread = tile row (output pixel) =====
    const int r_local = threadIdx.x;  // 0..127
    const uint32_t row_off = (r_local >> 3) * 1024 + (r_local & 7) * 128;
    const int sw = r_local & 7;
    int it = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      const int tm = tile % tiles_m, tn = tile / tiles_m;
      const int m = tm * 128 + r_local;
      const bool m_ok = m < M;
      int n = 0, ho = 0, wo = 0;
      if (m_ok) {
        n = m / (sh.Ho * sh.Wo);
        const int rem = m - n * sh.Ho * sh.Wo;
        ho = rem / sh.Wo;
        wo = rem - ho * sh.Wo;
      }
      const int hi0 = ho * sh.stride - sh.pad, wi0 = wo * sh.stride - sh.pad;
      const act_t* xn = x + (int64_t)n * sh.H * sh.W * sh.C;
      for (int kb = 0; kb < num_kb; ++kb, ++it) {
        const int s = it % STAGES;
        const uint32_t round = it / STAGES;
        mbar_wait_sleep(&empty[s], (round & 1) ^ 1);
        const uint32_t sa = smem_u32(smem + s * L::STAGE_BYTES) + row_off;
        if (threadIdx.x == 0) {
          mbar_expect_tx(&full[s], L::B_BYTES);
          tma_load_2d(smem + s * L::STAGE_BYTES + L::A_BYTES, &map_w, &full[s], kb * 64, tn * BN);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int k = kb * 64 + j * 8;
          const int tap = k / sh.C, c0 = k - tap * sh.C;
          const int rr = tap / sh.S, ss = tap - rr * sh.S;
          const int hi = hi0 + rr, wi = wi0 + ss;
          const bool ok = m_ok && tap < sh.R * sh.S && hi >= 0 && hi < sh.H && wi >= 0 && wi < sh.W;
          const act_t* src = ok ? xn + ((int64_t)hi * sh.W + wi) * sh.C + c0 : x;
          cp_async_16(sa + ((j ^ sw) << 4), src, ok);
        }
        cp_async_commit();
        if (it >= kLag) {
          cp_async_wait<kLag>();
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_arrive(&full[(it - kLag) % STAGES]);
        }
      }
    }
    // drain the last kLag stages
    cp_async_wait<0>();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    for (int d = (it >= kLag ? it - kLag : 0); d < it; ++d) mbar_arrive(&full[d % STAGES]);
  } else if (warp == kConvProdWarps) {
    // ===== MMA issuer: the warp runs the loop, one elected lane issues =====
    {
      // The issuer is one dependent instruction stream: at ~64 tensor cycles per MMA
      // a k-block's 4 MMAs last ~256 cycles, so its bookkeeping must stay well below
      // that.  Stage index / phase advance incrementally (no runtime % and /), the
      // operand descriptors are base + constant offsets (the 14-bit start-address
      // field never carries: smem < 256 KB), the centre-tap range is precomputed.
      constexpr uint32_t idesc = idesc_act_f32(128, BN);
      int t = 0, s = 0, dsl = 0;
      uint32_t ph = 0, dph = 0;
      if (b_loaded) mbar_wait(b_full, 0);   // also when the count leaves no tile: drain
      SkSched sc(ep.sk.enabled, num_tiles, num_kb, blockIdx.x, gridDim.x);
      SkWork w;
      const uint64_t a_desc0 = MODE == 2 ? sdesc_k_sw32(smem_u32(smem)) : sdesc_k_sw128(smem_u32(smem));
      const uint64_t b_desc0 = sdesc_k_sw128(smem_u32(sh.bres ? bres : smem + L::A_BYTES));
      const uint64_t ds_desc0 = sdesc_k_sw128(smem_u32(ds_ring));
      constexpr uint64_t kStageD = (uint64_t)(L::STAGE_BYTES >> 4), kBD = (uint64_t)(L::B_BYTES >> 4);
      const int cbl = sh.C / 64;
      const int kb_c0 = ((sh.R * sh.S) / 2) * cbl, kb_c1 = kb_c0 + cbl;   // DS: centre-tap k-blocks
      for (; sc.next(w); ++t) {
        const int acc = t & 1;
        const uint32_t use = t >> 1;
        mbar_wait(&acc_empty[acc], (use & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * NACC_COLS;
        for (int kb = w.kb0; kb < w.kb1; ++kb) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint64_t ad = a_desc0 + (uint64_t)s * kStageD;
          const uint64_t bd = sh.bres ? b_desc0 + (uint64_t)kb * kBD : b_desc0 + (uint64_t)s * kStageD;
          const bool ctr = DS && kb >= kb_c0 && kb < kb_c1;   // centre tap: downsample MMAs too
          if (ctr) {
            mbar_wait(&ds_full[dsl], dph);
            tc_fence_after();
          }
          if (elect_one_sync()) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              umma_bf16(d_tmem, ad + (uint64_t)(MODE == 2 ? kk * 256 : kk * 2), bd + (uint64_t)(kk * 2), idesc,
                        (kb != w.kb0 || kk != 0));
            if constexpr (DS) {
              if (ctr) {   // downsample accumulator: K = Cin (centre tap only)
                const uint64_t dd = ds_desc0 + (uint64_t)dsl * kBD;
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                  umma_bf16(d_tmem + BN, ad + (uint64_t)(kk * 2), dd + (uint64_t)(kk * 2), idesc,
                            kb != kb_c0 || kk != 0);
                umma_commit(&ds_empty[dsl]);
              }
            }
            umma_commit(&empty[s]);
          }
          __syncwarp();
          if (ctr && ++dsl == 2) {
            dsl = 0;
            dph ^= 1;
          }
          if (++s == nst) {
            s = 0;
            ph ^= 1;
          }
        }
        if (elect_one_sync()) umma_commit(&acc_full[acc]);
        __syncwarp();
      }
    }
  } else {
    // ===== epilogue =====
    const int quarter = warp & 3;
    const int chalf = (warp - kConvProdWarps - 1) >> 2;   // DS: column half of this warp
    int t = 0;
    SkSched sc(ep.sk.enabled, num_tiles, num_kb, blockIdx.x, gridDim.x);
    SkWork w;
    for (; sc.next(w); ++t) {
      const int tm = w.tile % tiles_m, tn = w.tile / tiles_m;
      const int acc = t & 1;
      mbar_wait_sleep(&acc_full[acc], (t >> 1) & 1);
      tc_fence_after();
      const uint32_t tacc0 = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * NACC_COLS;
      const uint32_t tacc = tacc0;
      const bool partial = w.kb0 != 0 || w.kb1 != num_kb;
      SkFix fx;
      if (partial) {   // stream-K: the last arriving segment reduces and stores the tile
        auto load32 = [&](int c, float (&v)[32]) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(tacc + c, r);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
        };
        if (!sk_arrive<BN>(ep.sk, sc, w, warp - kConvProdWarps - 1, 4, lane, fx, load32)) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&acc_empty[acc]);
          continue;
        }
      }
      const int m = tm * 128 + quarter * 32 + lane;
      const bool ok = m < M;
      int64_t oidx = m;   // output row: dense, zero-bordered [Ho+2, Wo+2], or shared-border
      if (ep.out_pad) {
        const int n = m / (sh.Ho * sh.Wo), rem = m - (m / (sh.Ho * sh.Wo)) * sh.Ho * sh.Wo;
        const int ho = rem / sh.Wo, wo = rem - (rem / sh.Wo) * sh.Wo;
        oidx = ep.out_pad == 2
                   ? (int64_t)(sh.Wo + 2) + ((int64_t)n * (sh.Ho + 1) + ho) * (sh.Wo + 1) + wo   // [Wo+2 margin][N, Ho+1, Wo+1]
                   : ((int64_t)n * (sh.Ho + 2) + ho + 1) * (sh.Wo + 2) + wo + 1;
      }
#pragma unroll 1
      for (int cc = DS ? chalf * BN : 0; cc < (DS ? (chalf + 1) * BN : BN); cc += 32) {
        // DS: columns [BN, 2 BN) of the buffer are the downsample accumulator
        const bool dsp = DS && cc >= BN;
        const int c = dsp ? cc - BN : cc;
        act_t* yout = dsp ? ep.y_ds : ep.y;
        const float* bvec = dsp ? ep.bias_ds : ep.bias;
        uint32_t r[32];
        tmem_ld_32x32b_x32(tacc + cc, r);
        tmem_ld_wait();
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
        if (partial) sk_sum<BN>(ep.sk, sc, w, warp - kConvProdWarps - 1, 4, lane, fx, c, v);
        if (!ok) continue;
        const int col0 = tn * BN + c;
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          const float4 b = __ldg(reinterpret_cast<const float4*>(bvec + col0 + i));
          v[i] += b.x;
          v[i + 1] += b.y;
          v[i + 2] += b.z;
          v[i + 3] += b.w;
        }
        if (ep.residual && !dsp) {
          const uint4* rp = reinterpret_cast<const uint4*>(ep.residual + oidx * sh.Cout + col0);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint4 u = __ldg(rp + q);
            const act2_t* h2 = reinterpret_cast<const act2_t*>(&u);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 f = act2_to_float2(h2[e]);
              v[q * 8 + 2 * e] += f.x;
              v[q * 8 + 2 * e + 1] += f.y;
            }
          }
        }
        if (ep.relu && !dsp) {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = fmaxf(v[i], 0.0f);
        }
        uint4* dp = reinterpret_cast<uint4*>(yout + oidx * sh.Cout + col0);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 u;
          u.x = pack_act(v[q * 8 + 0], v[q * 8 + 1]);
          u.y = pack_act(v[q * 8 + 2], v[q * 8 + 3]);
          u.z = pack_act(v[q * 8 + 4], v[q * 8 + 5]);
          u.w = pack_act(v[q * 8 + 6], v[q * 8 + 7]);
          dp[q] = u;
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[acc]);
    }
  }
  __syncthreads();
  if (warp == kConvProdWarps) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 2 * NACC_COLS);
  }
}

template <int BN, int STAGES, int MODE, bool DS = false>
static int launch_conv(const act_t* x, const CUtensorMap& mw, const CUtensorMap& mx,
                       const ConvShape& sh, const ConvEpi& ep, cudaStream_t s,
                       const CUtensorMap* mwds = nullptr) {
  using L = ConvSmem<BN, STAGES, DS>;
  auto kern = conv_bf16_tcgen05<BN, STAGES, MODE, DS>;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024) != cudaSuccess)
      return GG_ERR_CUDA;
    attr = true;
  }
  const int tiles = ((sh.M + 127) / 128) * (sh.Cout / BN);
  const int grid = ep.sk.enabled ? num_sms() : (tiles < num_sms() ? tiles : num_sms());
  const int smem = sh.bres ? sh.bres_stages * L::STAGE_BYTES + (sh.Kpad / 64) * L::B_BYTES + 256 + 1024
                           : L::TOTAL;
  if (launch_pdl(kern, dim3(grid), dim3(32 * (kConvProdWarps + 1 + conv_epi_warps(DS))), smem, s, x, mw, mx,
                 mwds ? *mwds : mw, sh, ep) !=
      cudaSuccess)
    return GG_ERR_CUDA;
  return GG_OK;
}

// TMA im2col map over an NHWC bf16 activation: 128 output pixels x 64 channels per load.
static PFN_cuTensorMapEncodeIm2col_v12000 g_encode_im2col = nullptr;
static int make_map_im2col(CUtensorMap* map, const void* x, const ConvShape& sh, int cpb) {
  if (!g_encode_im2col) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return GG_ERR_CUDA;
    g_encode_im2col = reinterpret_cast<PFN_cuTensorMapEncodeIm2col_v12000>(fn);
  }
  cuuint64_t dims[4] = {(cuuint64_t)sh.C, (cuuint64_t)sh.W, (cuuint64_t)sh.H, (cuuint64_t)sh.N};
  cuuint64_t strides[3] = {(cuuint64_t)sh.C * 2, (cuuint64_t)sh.W * sh.C * 2,
                           (cuuint64_t)sh.H * sh.W * sh.C * 2};
  // traversal box of the receptive-field origin: [-pad, W + pad - S] (CUTLASS fprop convention)
  int lower[2] = {-sh.pad, -sh.pad};
  int upper[2] = {sh.pad_hi - (sh.S - 1), sh.pad_hi - (sh.R - 1)};
  cuuint32_t estr[4] = {1, (cuuint32_t)sh.stride, (cuuint32_t)sh.stride, 1};
  CUresult r = g_encode_im2col(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, const_cast<void*>(x), dims,
                               strides, lower, upper, (cuuint32_t)cpb, 128, estr,
                               CU_TENSOR_MAP_INTERLEAVE_NONE,
                               cpb == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_32B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? GG_OK : GG_ERR_INVALID_ARGUMENT;
}

// ---- pooling / layout kernels (HBM-bound) -----------------------------------
// NCHW fp32 image -> NHWC bf16 with channels zero-padded to cpad.
__global__ void nchw_to_nhwc_pad(const float* __restrict__ in, act_t* __restrict__ out,
                                 int N, int C, int H, int W, int cpad) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // pixel
  if (p >= (int64_t)N * H * W) return;
  const int n = p / (H * W);
  const int hw = p - (int64_t)n * H * W;
  __align__(16) act_t v[8];
  for (int c0 = 0; c0 < cpad; c0 += 8) {
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int c = c0 + e;
      v[e] = float2act(c < C ? __ldg(in + ((int64_t)n * C + c) * H * W + hw) : 0.0f);
    }
    *reinterpret_cast<uint4*>(out + p * cpad + c0) = *reinterpret_cast<uint4*>(v);
  }
}

// 3x3 stride-2 pad-1 max pool, NHWC, 8 channels per thread.
__global__ void maxpool3x3s2(const act_t* __restrict__ in, act_t* __restrict__ out,
                             int N, int H, int W, int C, int Ho, int Wo, const int32_t* count,
                             int out_pad) {
  griddep_wait();
  griddep_launch();
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int cg = C / 8;
  if (count) N = min(N, __ldg(count));
  if (idx >= (int64_t)N * Ho * Wo * cg) return;
  const int c0 = (idx % cg) * 8;
  const int64_t p = idx / cg;
  const int wo = p % Wo, ho = (p / Wo) % Ho, n = p / ((int64_t)Wo * Ho);
  float m[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) m[e] = -INFINITY;
  for (int r = 0; r < 3; ++r) {
    const int hi = ho * 2 - 1 + r;
    if (hi < 0 || hi >= H) continue;
    for (int s = 0; s < 3; ++s) {
      const int wi = wo * 2 - 1 + s;
      if (wi < 0 || wi >= W) continue;
      const uint4 u = __ldg(reinterpret_cast<const uint4*>(in + (((int64_t)n * H + hi) * W + wi) * C + c0));
      const act2_t* h2 = reinterpret_cast<const act2_t*>(&u);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = act2_to_float2(h2[e]);
        m[2 * e] = fmaxf(m[2 * e], f.x);
        m[2 * e + 1] = fmaxf(m[2 * e + 1], f.y);
      }
    }
  }
  uint4 u;
  u.x = pack_act(m[0], m[1]);
  u.y = pack_act(m[2], m[3]);
  u.z = pack_act(m[4], m[5]);
  u.w = pack_act(m[6], m[7]);
  const int64_t o = out_pad ? ((int64_t)n * (Ho + 2) + ho + 1) * (Wo + 2) + wo + 1 : p;
  *reinterpret_cast<uint4*>(out + o * C + c0) = u;
}

// 3x3 stride-2 pad-1 max pool, blocked: a thread owns 8 channels of a 4 x 2
// block of outputs and reads its 9 x 5 input window once (45 16-byte loads for
// 8 outputs instead of 72), maxing packed bf16x2 directly (exact).  Threads of
// a warp: 8 channel groups x 4 column pairs, so every load instruction touches
// four 128-byte pixel rows.
constexpr int kPoolRows = 4, kPoolCols = 2;
__global__ void __launch_bounds__(256) maxpool3x3s2_blocked(const act_t* __restrict__ in,
                                                            act_t* __restrict__ out, int N,
                                                            int H, int W, int C, int Ho, int Wo,
                                                            const int32_t* count, int out_pad) {
  griddep_wait();
  griddep_launch();
  const int cg = C / 8;
  const int wb = (Wo + kPoolCols - 1) / kPoolCols, hb = (Ho + kPoolRows - 1) / kPoolRows;
  if (count) N = min(N, __ldg(count));
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)N * hb * wb * cg) return;
  const int c0 = (int)(idx % cg) * 8;
  idx /= cg;
  const int bw = (int)(idx % wb);
  idx /= wb;
  const int bh = (int)(idx % hb);
  const int n = (int)(idx / hb);
  const int ho0 = bh * kPoolRows, wo0 = bw * kPoolCols;
  const act2_t ninf = float2act2(-INFINITY);
  act2_t m[kPoolRows][kPoolCols][4];
#pragma unroll
  for (int i = 0; i < kPoolRows; ++i)
#pragma unroll
    for (int j = 0; j < kPoolCols; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) m[i][j][e] = ninf;
  const act_t* img = in + (int64_t)n * H * W * C + c0;
  const uint64_t pol = l2_policy_evict_first();   // single-use input (kept in L2 by the stem)
#pragma unroll
  for (int r = 0; r < 2 * kPoolRows + 1; ++r) {
    const int hi = 2 * ho0 - 1 + r;
    if (hi < 0 || hi >= H) continue;
#pragma unroll
    for (int q = 0; q < 2 * kPoolCols + 1; ++q) {
      const int wi = 2 * wo0 - 1 + q;
      if (wi < 0 || wi >= W) continue;
      const uint4 u = ld_global_nc_v4_hint(img + ((int64_t)hi * W + wi) * C, pol);
      const act2_t* v = reinterpret_cast<const act2_t*>(&u);
      // input row r feeds output rows i with 2i <= r <= 2i + 2; column q feeds j with 2j <= q <= 2j + 2
#pragma unroll
      for (int i = 0; i < kPoolRows; ++i) {
        if (r < 2 * i || r > 2 * i + 2) continue;
#pragma unroll
        for (int j = 0; j < kPoolCols; ++j) {
          if (q < 2 * j || q > 2 * j + 2) continue;
#pragma unroll
          for (int e = 0; e < 4; ++e) m[i][j][e] = __hmax2(m[i][j][e], v[e]);
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < kPoolRows; ++i) {
    const int ho = ho0 + i;
    if (ho >= Ho) break;
#pragma unroll
    for (int j = 0; j < kPoolCols; ++j) {
      const int wo = wo0 + j;
      if (wo >= Wo) break;
      const int64_t o = out_pad == 2   // shared-border layout: (Wo+2)-row margin, [Ho+1, Wo+1] images
                            ? (int64_t)(Wo + 2) + ((int64_t)n * (Ho + 1) + ho) * (Wo + 1) + wo
                        : out_pad ? ((int64_t)n * (Ho + 2) + ho + 1) * (Wo + 2) + wo + 1
                                : ((int64_t)n * Ho + ho) * Wo + wo;
      *reinterpret_cast<uint4*>(out + o * C + c0) = *reinterpret_cast<const uint4*>(m[i][j]);
    }
  }
}

// Global average pool NHWC [N, HW, C] -> [N, C] bf16 (fp32 sum).  Block =
// (image, 64 channels): warp w owns channels 8w..8w+7 (one 16-byte load per
// pixel), its lanes stride over the pixels, then a warp reduction.
__global__ void __launch_bounds__(256) avgpool_global(const act_t* __restrict__ in,
                                                      act_t* __restrict__ out, int N,
                                                      int HW, int C, const int32_t* count,
                                                      int denom) {
  griddep_wait();
  griddep_launch();
  if (count) N = min(N, __ldg(count));
  const int n = blockIdx.y;
  if (n >= N) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c0 = blockIdx.x * 64 + warp * 8;
  float s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const act_t* base = in + (int64_t)n * HW * C + c0;
  for (int p = lane; p < HW; p += 32) {
    const uint4 u = __ldg(reinterpret_cast<const uint4*>(base + (int64_t)p * C));
    const act2_t* h2 = reinterpret_cast<const act2_t*>(&u);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = act2_to_float2(h2[e]);
      s[2 * e] += f.x;
      s[2 * e + 1] += f.y;
    }
  }
#pragma unroll
  for (int e = 0; e < 8; ++e)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s[e] += __shfl_xor_sync(0xffffffffu, s[e], o);
  if (lane == 0) {
    const float inv = 1.0f / (denom > 0 ? denom : HW);   // padded input: borders are zeros
    uint4 u;
    u.x = pack_act(s[0] * inv, s[1] * inv);
    u.y = pack_act(s[2] * inv, s[3] * inv);
    u.z = pack_act(s[4] * inv, s[5] * inv);
    u.w = pack_act(s[6] * inv, s[7] * inv);
    *reinterpret_cast<uint4*>(out + (int64_t)n * C + c0) = u;
  }
}

// Global average pool to fp32 [N, C] (same traversal as avgpool_global, no
// bf16 rounding of the pooled vector: the head stays in fp32).
__global__ void __launch_bounds__(256) avgpool_global_f32(const act_t* __restrict__ in,
                                                          float* __restrict__ out, int N, int HW,
                                                          int C, const int32_t* count, int denom) {
  griddep_wait();
  griddep_launch();
  if (count) N = min(N, __ldg(count));
  const int n = blockIdx.y;
  if (n >= N) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c0 = blockIdx.x * 64 + warp * 8;
  float s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const act_t* base = in + (int64_t)n * HW * C + c0;
  for (int p = lane; p < HW; p += 32) {
    const uint4 u = __ldg(reinterpret_cast<const uint4*>(base + (int64_t)p * C));
    const act2_t* h2 = reinterpret_cast<const act2_t*>(&u);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = act2_to_float2(h2[e]);
      s[2 * e] += f.x;
      s[2 * e + 1] += f.y;
    }
  }
#pragma unroll
  for (int e = 0; e < 8; ++e)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s[e] += __shfl_xor_sync(0xffffffffu, s[e], o);
  if (lane == 0) {
    const float inv = 1.0f / (denom > 0 ? denom : HW);
    float4* o4 = reinterpret_cast<float4*>(out + (int64_t)n * C + c0);
    o4[0] = make_float4(s[0] * inv, s[1] * inv, s[2] * inv, s[3] * inv);
    o4[1] = make_float4(s[4] * inv, s[5] * inv, s[6] * inv, s[7] * inv);
  }
}

// fp32 classifier head: logits[n, j] = pooled[n, :] . w[j, :] + b[j] for the
// first *count images.  Block = (kFcCls classes, kFcImg images), one warp per
// image: the classes' weight rows are staged in smem once per block (before the
// PDL wait), each lane takes a C / 32 slice of the image row (coalesced float4
// loads) against the kFcCls rows (conflict-free float4 LDS), then one
// butterfly reduction per class.  ~1000 small blocks: the head is latency-
// bound, so parallelism beats reuse here.
constexpr int kFcCls = 8;
constexpr int kFcImg = 8;
__global__ void __launch_bounds__(32 * kFcImg) fc_f32_kernel(const float* __restrict__ pooled,
                                                            const float* __restrict__ w,
                                                            const float* __restrict__ b, int N, int C,
                                                            int ncls, float* __restrict__ logits,
                                                            int64_t ldl, const int32_t* count) {
  extern __shared__ __align__(16) float ws[];   // [kFcCls][C]
  const int j0 = blockIdx.x * kFcCls;
  const int nc = min(kFcCls, ncls - j0);
  const int c4 = C / 4;
  for (int e0 = threadIdx.x; e0 < kFcCls * c4; e0 += 4 * blockDim.x) {
    float4 v[4];   // four loads in flight before the stores
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = e0 + u * blockDim.x, c = e / c4, k = e - c * c4;
      v[u] = (e < kFcCls * c4 && c < nc)
                 ? __ldg(reinterpret_cast<const float4*>(w + (int64_t)(j0 + c) * C) + k)
                 : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = e0 + u * blockDim.x;
      if (e < kFcCls * c4) reinterpret_cast<float4*>(ws)[e] = v[u];
    }
  }
  griddep_wait();
  griddep_launch();
  if (count) N = min(N, __ldg(count));
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.y * kFcImg + (threadIdx.x >> 5);
  if (i >= N) return;
  const float4* x4 = reinterpret_cast<const float4*>(pooled + (int64_t)i * C);
  float acc[kFcCls];
#pragma unroll
  for (int c = 0; c < kFcCls; ++c) acc[c] = 0.f;
  for (int f = lane; f < c4; f += 32) {
    const float4 x = __ldg(x4 + f);
#pragma unroll
    for (int c = 0; c < kFcCls; ++c) {
      const float4 v = reinterpret_cast<const float4*>(ws + c * C)[f];
      acc[c] = fmaf(x.w, v.w, fmaf(x.z, v.z, fmaf(x.y, v.y, fmaf(x.x, v.x, acc[c]))));
    }
  }
#pragma unroll
  for (int c = 0; c < kFcCls; ++c)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], o);
  if (lane < nc) {
    float r = acc[0];
#pragma unroll
    for (int c = 1; c < kFcCls; ++c) r = lane == c ? acc[c] : r;
    logits[(int64_t)i * ldl + j0 + lane] = r + __ldg(b + j0 + lane);
  }
}

}  // namespace gg

using namespace gg;

extern "C" int gg_avgpool_fc(const void* x, int32_t N, int32_t HW, int32_t C, int32_t denom,
                             const float* w_fc, const float* b_fc, int32_t ncls, float* pooled,
                             float* logits, int64_t ld_logits, const int32_t* count_dev,
                             void* stream) {
  if (!x || !w_fc || !b_fc || !pooled || !logits || N < 1 || ncls < 1 || denom < 0 ||
      ld_logits < ncls)
    return GG_ERR_INVALID_ARGUMENT;
  if (C % 128 || C > 1536 || N > 65535 * kFcImg) return GG_ERR_UNSUPPORTED;
  if (launch_pdl(avgpool_global_f32, dim3((unsigned)(C / 64), (unsigned)N), dim3(256), 0,
                 gg_stream(stream), reinterpret_cast<const act_t*>(x), pooled, N, HW, C,
                 count_dev, denom) != cudaSuccess)
    return GG_ERR_CUDA;
  if (launch_pdl(fc_f32_kernel,
                 dim3((unsigned)((ncls + kFcCls - 1) / kFcCls), (unsigned)((N + kFcImg - 1) / kFcImg)),
                 dim3(32 * kFcImg), (size_t)kFcCls * C * 4, gg_stream(stream),
                 (const float*)pooled, w_fc, b_fc, N, C, ncls, logits, ld_logits, count_dev) != cudaSuccess)
    return GG_ERR_CUDA;
  GG_LAUNCH_OK();
  return GG_OK;
}

extern "C" int gg_conv2d(const void* x, int32_t N, int32_t H, int32_t W, int32_t C, const void* w,
                         int32_t Cout, int32_t R, int32_t S, int32_t stride, int32_t pad,
                         int32_t Kpad, const float* bias, const void* residual, int32_t relu,
                         void* y, int32_t pad_hi, int32_t out_pad, const int32_t* count_dev,
                         void* stream) {
  if (!x || !w || !y || !bias || N <= 0 || H <= 0 || W <= 0 || R <= 0 || S <= 0 || stride <= 0)
    return GG_ERR_INVALID_ARGUMENT;
  // pad may be negative (-1): reading the interior of an already zero-padded input
  if (C % 8 || Kpad % 64 || Kpad < R * S * C || Cout % 64 || pad < -1) return GG_ERR_UNSUPPORTED;
  ConvShape sh;
  sh.N = N; sh.H = H; sh.W = W; sh.C = C; sh.Cout = Cout;
  sh.R = R; sh.S = S; sh.stride = stride; sh.pad = pad; sh.Kpad = Kpad;
  sh.pad_hi = pad_hi < 0 ? pad : pad_hi;
  sh.bres = 0;
  sh.bres_stages = 0;
  sh.Ho = (H + pad + sh.pad_hi - R) / stride + 1;
  sh.Wo = (W + pad + sh.pad_hi - S) / stride + 1;
  const int64_t M = (int64_t)N * sh.Ho * sh.Wo;
  if (M > 0x7fffffff) return GG_ERR_UNSUPPORTED;
  sh.M = (int)M;
  ConvEpi ep{reinterpret_cast<act_t*>(y), bias,
             reinterpret_cast<const act_t*>(residual), relu, count_dev, out_pad,
             StreamK{nullptr, nullptr, 0}, nullptr, nullptr};
  // N tile: minimize the larger of (tensor time of the busiest SM) and (operand
  // bytes streamed from L2: every tile re-reads its A rows and its B columns per
  // k-block).  Measured on B200: ~8 TB/s of TMA operand traffic, MMA 128xBN x K16
  // in BN/2 cycles.  Small-M late layers prefer wide tiles, layer1 (Cout 64) 64.
  const int64_t tiles_m = (M + 127) / 128;
  const int64_t nkb = Kpad / 64;
  int bn = 64;
  double best = 1e30;
  for (int cand : {64, 128, 256}) {
    if (cand > Cout || Cout % cand) continue;
    const int64_t tiles = tiles_m * (Cout / cand);
    const int64_t waves = (tiles + num_sms() - 1) / num_sms();
    const double t_mma = (double)waves * nkb * 2 * cand / 1.9e9;
    const double t_l2 = (double)tiles * nkb * (16384.0 + cand * 128.0) / 8.0e12;
    const double t = t_mma > t_l2 ? t_mma : t_l2;
    if (t < best * 0.97) {
      best = t;
      bn = cand;
    }
  }
  CUtensorMap mw, mx;
  int rc = make_map_2d(&mw, w, Cout, Kpad, Kpad, bn);
  if (rc) return rc;
  const int mode = (C % 64 == 0 && Kpad == R * S * C) ? 1
                   : (C == 16 && (R * S) % 4 == 0 && Kpad == R * S * C) ? 2 : 0;
  if (mode) {
    rc = make_map_im2col(&mx, x, sh, mode == 1 ? 64 : 16);
    if (rc) return rc;
    // resident weights when the whole N = Cout slab fits next to a 4-deep A ring
    const int stage_bytes = 128 * 128 + bn * 128;
    const int64_t need = 4LL * stage_bytes + (Kpad / 64) * (int64_t)bn * 128 + 1280;
    if (bn == Cout && need <= 227 * 1024) {
      sh.bres = 1;
      sh.bres_stages = 4;
    }
  } else {
    mx = mw;  // unused by the gather path
  }
  cudaStream_t s = gg_stream(stream);
  const act_t* xb = reinterpret_cast<const act_t*>(x);
  if (mode == 1 && streamk_wanted(tiles_m * (Cout / bn), nkb, num_sms())) {
    bool ok = false;
    StreamK sk = streamk_workspace(s, (int64_t)num_sms() * 2 * 128 * bn,
                                   tiles_m * (Cout / bn) * 4 * 2, ok);
    if (ok) ep.sk = sk;
  }
  if (mode == 1) {
    switch (bn) {
      case 256: return launch_conv<256, 4, 1>(xb, mw, mx, sh, ep, s);
      case 128: return launch_conv<128, 6, 1>(xb, mw, mx, sh, ep, s);
      default: return launch_conv<64, 8, 1>(xb, mw, mx, sh, ep, s);
    }
  }
  if (mode == 2) {
    switch (bn) {
      case 256: return launch_conv<256, 4, 2>(xb, mw, mx, sh, ep, s);
      case 128: return launch_conv<128, 6, 2>(xb, mw, mx, sh, ep, s);
      default: return launch_conv<64, 8, 2>(xb, mw, mx, sh, ep, s);
    }
  }
  switch (bn) {
    case 256: return launch_conv<256, 4, 0>(xb, mw, mx, sh, ep, s);
    case 128: return launch_conv<128, 6, 0>(xb, mw, mx, sh, ep, s);
    default: return launch_conv<64, 8, 0>(xb, mw, mx, sh, ep, s);
  }
}

extern "C" int gg_conv2d_ds(const void* x, int32_t N, int32_t H, int32_t W, int32_t C, const void* w,
                            int32_t Cout, const float* bias, void* y, const void* w_ds,
                            const float* bias_ds, void* y_ds, int32_t in_shared, int32_t out_shared,
                            const int32_t* count_dev, void* stream) {
  // 3x3 / stride 2 (+ folded BN + ReLU) fused with the block's 1x1 / stride 2
  // downsample (+ folded BN, no ReLU) of the same input.  Input: zero-bordered
  // [N, H, W, C] (H, W padded extents, pad 0) or, in_shared, the shared-border
  // layout ([W+1 margin][N, H, W, C] with the image in [H-1, W-1]: pad 1 before, the
  // zero row / column after).  Outputs zero-bordered or (out_shared) shared-border.
  if (!x || !w || !y || !bias || !w_ds || !bias_ds || !y_ds || N <= 0 || H < 3 || W < 3)
    return GG_ERR_INVALID_ARGUMENT;
  if (C % 64 || Cout % 128) return GG_ERR_UNSUPPORTED;
  ConvShape sh;
  sh.N = N; sh.H = H; sh.W = W; sh.C = C; sh.Cout = Cout;
  sh.R = 3; sh.S = 3; sh.stride = 2; sh.pad = in_shared ? 1 : 0; sh.pad_hi = 0; sh.Kpad = 9 * C;
  sh.bres = 0;
  sh.bres_stages = 0;
  sh.Ho = (H + sh.pad - 3) / 2 + 1;
  sh.Wo = (W + sh.pad - 3) / 2 + 1;
  if (in_shared) x = reinterpret_cast<const act_t*>(x) + (int64_t)(W + 1) * C;   // past the margin
  const int64_t M = (int64_t)N * sh.Ho * sh.Wo;
  if (M > 0x7fffffff) return GG_ERR_UNSUPPORTED;
  sh.M = (int)M;
  ConvEpi ep{reinterpret_cast<act_t*>(y), bias, nullptr, 1, count_dev, out_shared ? 2 : 1,
             StreamK{nullptr, nullptr, 0}, reinterpret_cast<act_t*>(y_ds), bias_ds};
  constexpr int BN = 128;
  CUtensorMap mw, mwds, mx;
  int rc = make_map_2d(&mw, w, Cout, sh.Kpad, sh.Kpad, BN);
  if (!rc) rc = make_map_2d(&mwds, w_ds, Cout, C, C, BN);
  if (!rc) rc = make_map_im2col(&mx, x, sh, 64);
  if (rc) return rc;
  return launch_conv<BN, 6, 1, true>(reinterpret_cast<const act_t*>(x), mw, mx, sh, ep,
                                     gg_stream(stream), &mwds);
}

extern "C" int gg_nchw_to_nhwc(const float* x, int32_t N, int32_t C, int32_t H, int32_t W,
                               int32_t cpad, void* y, void* stream) {
  if (!x || !y || cpad % 8 || cpad < C) return GG_ERR_INVALID_ARGUMENT;
  const int64_t pixels = (int64_t)N * H * W;
  nchw_to_nhwc_pad<<<(unsigned)((pixels + 255) / 256), 256, 0, gg_stream(stream)>>>(
      x, reinterpret_cast<act_t*>(y), N, C, H, W, cpad);
  GG_LAUNCH_OK();
  return GG_OK;
}

extern "C" int gg_maxpool3x3s2(const void* x, int32_t N, int32_t H, int32_t W, int32_t C, void* y,
                               int32_t out_pad, const int32_t* count_dev, void* stream) {
  if (!x || !y || C % 8) return GG_ERR_INVALID_ARGUMENT;
  const int Ho = (H + 2 - 3) / 2 + 1, Wo = (W + 2 - 3) / 2 + 1;
  const int64_t work = (int64_t)N * ((Ho + kPoolRows - 1) / kPoolRows) *
                       ((Wo + kPoolCols - 1) / kPoolCols) * (C / 8);
  if (launch_pdl(maxpool3x3s2_blocked, dim3((unsigned)((work + 255) / 256)), dim3(256), 0, gg_stream(stream),
      reinterpret_cast<const act_t*>(x), reinterpret_cast<act_t*>(y), N, H, W, C,
      Ho, Wo, count_dev, out_pad) != cudaSuccess)
    return GG_ERR_CUDA;
  GG_LAUNCH_OK();
  return GG_OK;
}

extern "C" int gg_avgpool(const void* x, int32_t N, int32_t HW, int32_t C, void* y,
                          int32_t denom, const int32_t* count_dev, void* stream) {
  if (!x || !y || C % 8 || denom < 0 || N < 1) return GG_ERR_INVALID_ARGUMENT;
  if (C % 64 || N > 65535) return GG_ERR_UNSUPPORTED;
  if (launch_pdl(avgpool_global, dim3((unsigned)(C / 64), (unsigned)N), dim3(256), 0, gg_stream(stream),
      reinterpret_cast<const act_t*>(x), reinterpret_cast<act_t*>(y), N, HW, C,
      count_dev, denom) != cudaSuccess)
    return GG_ERR_CUDA;
  GG_LAUNCH_OK();
  return GG_OK;
}
