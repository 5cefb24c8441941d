// gg_conv_span.cu — stride-1 convolutions on zero-padded NHWC activations with
// ONE operand load per tile for all taps ("span" convolution).
//
// Activations live padded: [N, Hp, Wp, C] with zero borders.  Index output
// positions in the padded input space, m = (n*Hp + h)*Wp + w; tap (r, s) of
// output m reads padded pixel m + r*Wp + s — a uniform shift.  So for a tile
// of 128 consecutive m, the RT x RT A operands are shifted views of ONE span of
// 128 + (RT-1)*(Wp+1) pixel rows, loaded once per channel block by TMA
// (instead of RT*RT im2col loads).  The span sits in shared memory in the
// K-major swizzled layout (CH = 64 channels: 128-B rows, SWIZZLE_128B; CH = 16:
// 32-B rows, SWIZZLE_32B); a shift by one pixel is +row bytes on the UMMA
// descriptor start address — the hardware applies the swizzle XOR to absolute
// address bits, so row starts inside a swizzle atom need no base offset
// (verified by tests/test_conv_span_gpu.py).
//
// Two instantiations serve ResNet-18:
//   * 3x3 / 1, pad 1, C % 64 == 0 (layers 1-4): output written padded in the
//     same geometry at m + Wp + 1; positions with h >= H or w >= W are written
//     as ZEROS — they land exactly on the output's padding, so the next layer
//     reads correct zero borders.
//   * the stem: 7x7 / 2 on the image = 4x4 / 1 over its space-to-depth(2)
//     (16 channels), input padded 2 before / 1 after; output dense (positions
//     outside the real 112 x 112 grid are skipped).
//
// Roles (persistent CTAs, one per SM):
//   warp 0      TMA producer: A spans (ring of as many stages as fit) and B
//               (the whole BN x K weight slab once per CTA when it fits, else
//               a ring of one tap slab per stage)
//   warp 1      TMEM allocator + tcgen05.mma issuer.  The issue loop is lean —
//               descriptors are base + offsets, all taps unrolled — because at
//               N = 64 the tensor pipe takes a new MMA every 32-48 cycles
//               (tools/mma_bench.cu: a naive loop issues one per ~90 cycles)
//   warps 2..9  epilogue: tcgen05.ld, folded-BN bias, residual, ReLU, bf16;
//               two column halves x four TMEM lane quarters
#include <cudaTypedefs.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "gg_common.cuh"
#include "gg_kernels.h"
#include "gg_streamk.cuh"
#include "gg_tc.cuh"
#include "gg_act.cuh"

namespace gg {
using namespace tc;

constexpr int kSpanMaxStages = 16;
constexpr int kSpanEpiWarps = 8;
constexpr int kSpanThreads = 64 + 32 * kSpanEpiWarps;
constexpr int kSpanSmemMax = 227 * 1024;
constexpr int kSpanStgBytes = 8 * 4096 + 2048;   // pair TMA epilogue staging (+ alignment)

struct SpanShape {
  int N, H, W, C, Cout;
  int Hp, Wp;          // padded input extents
  int Ho, Wo;          // real output extents (dense mode: output row pitch)
  int span_rows;       // 128 + (RT-1)*(Wp+1)
  int box_rows, boxes; // the span as `boxes` TMA boxes of box_rows (<= 256) rows
  int a_stage_bytes;   // boxes * box_rows * row bytes, rounded up to 1 KB
  int a_stages;
  int b_stages;        // ring depth (ignored when bres)
  int bres;            // whole weight slab resident
};

struct SpanEpi {
  act_t* y;
  const float* bias;
  const act_t* residual;  // padded, same geometry as y (padded mode), or null
  int relu;
  const int32_t* count;
  unsigned long long* prof;   // debug (GG_SPAN_PROF): per-CTA globaltimer start / end
  const act_t* x16;   // CH == 16: the pre-swizzled input (bulk-copied)
  int nostore;                // debug (GG_SPAN_NOSTORE): skip the output stores
  int tma_out;                // pair kernel, padded mode: outputs / residuals via smem + TMA
  StreamK sk;                 // pair kernel: stream-K over (pair tile, channel block), or disabled
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint64_t sdesc_sw(uint32_t addr, int row_bytes) {
  return row_bytes == 128 ? sdesc_k_sw128(addr) : sdesc_k_sw32(addr);
}

template <int BN, int CH, int RT, bool DENSE, int MT>
__global__ void __launch_bounds__(kSpanThreads, 1)
    conv_span_tcgen05(const __grid_constant__ CUtensorMap map_x,
                      const __grid_constant__ CUtensorMap map_w, const __grid_constant__ CUtensorMap map_out,
                      const __grid_constant__ CUtensorMap map_res, SpanShape sh, SpanEpi ep) {
  constexpr int RB = CH * 2;                 // bytes per pixel row (one swizzle row)
  constexpr int KSTEPS = CH / 16;            // MMAs per tap
  constexpr int TAPS = RT * RT;
  constexpr int B_BYTES = BN * RB;           // one tap slab of B
  constexpr int BM = 128 * MT;               // MT M=128 sub-tiles share every B slab
  constexpr int ACC_COLS = MT * BN;          // TMEM columns per accumulator buffer
  // accumulator buffers in TMEM: 4 when they fit (N = 64 tiles are short — 9
  // taps x 4 MMAs — so two buffers let one slow epilogue stall the tensor pipe)
  constexpr int NACC = 512 / ACC_COLS >= 4 ? 4 : 2;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_align1k(smem_raw);
  const int cblocks = sh.C / CH;
  const int nkb = cblocks * TAPS;
  const int AST = sh.a_stages, BST = sh.b_stages;
  uint8_t* a_base = smem;
  uint8_t* b_base = smem + AST * sh.a_stage_bytes;
  const int b_slots = sh.bres ? nkb : BST;
  uint64_t* bars = reinterpret_cast<uint64_t*>(b_base + b_slots * B_BYTES);
  uint64_t* a_full = bars;
  uint64_t* a_empty = a_full + kSpanMaxStages;
  uint64_t* b_full = a_empty + kSpanMaxStages;
  uint64_t* b_empty = b_full + kSpanMaxStages;
  uint64_t* acc_full = b_empty + kSpanMaxStages;
  uint64_t* acc_empty = acc_full + NACC;
  uint64_t* bres_full = acc_empty + NACC;
  uint64_t* res_full = bres_full + 1;      // [8 warps][2]: residual boxes landed (TMA epilogue)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(res_full + 2 * kSpanEpiWarps);
  uint8_t* stg_base = smem_align1k(reinterpret_cast<uint8_t*>(bars) + 1024);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (ep.prof && threadIdx.x == 0) {
    ep.prof[2 * blockIdx.x] = gtimer();
    ep.prof[2048 + 2 * blockIdx.x] = clock64();
  }
  griddep_launch();   // the successor may begin its prologue as SMs free up
  const int img = sh.Hp * sh.Wp;
  const int tiles_n = sh.Cout / BN;

  if (threadIdx.x == 0) {
    for (int i = 0; i < AST; ++i) {   // only the ring slots this launch uses
      mbar_init(&a_full[i], 1);
      mbar_init(&a_empty[i], 1);
    }
    for (int i = 0; i < BST; ++i) {
      mbar_init(&b_full[i], 1);
      mbar_init(&b_empty[i], 1);
    }
    for (int i = 0; i < NACC; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], kSpanEpiWarps);
    }
    mbar_init(bres_full, 1);
    for (int i = 0; i < 2 * kSpanEpiWarps; ++i) mbar_init(&res_full[i], 1);
    fence_mbar_init();
    tma_prefetch(&map_x);
    tma_prefetch(&map_w);
    if (ep.tma_out) {
      tma_prefetch(&map_out);
      if (ep.residual) tma_prefetch(&map_res);
    }
  }
  if (warp == 1) tmem_alloc(tmem_slot, NACC * ACC_COLS);
  // the weight slab does not depend on the predecessor: start it before the wait
  if (warp == 0 && lane == 0 && sh.bres) {
    const int tiles_max = (sh.N * img + BM - 1) / BM * tiles_n;
    if (tiles_max > (int)blockIdx.x) {
      mbar_expect_tx(bres_full, nkb * B_BYTES);
      for (int kb = 0; kb < nkb; ++kb) tma_load_2d(b_base + kb * B_BYTES, &map_w, bres_full, kb * CH, 0);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  griddep_wait();   // activations, residual, count and output all follow the predecessor
  const int n_eff = ep.count ? min(sh.N, __ldg(ep.count)) : sh.N;
  const int Mtot = n_eff * img;
  const int tiles_m = (Mtot + BM - 1) / BM;
  const int num_tiles = tiles_m * tiles_n;
  const bool b_loaded = sh.bres && (sh.N * img + BM - 1) / BM * tiles_n > (int)blockIdx.x;

  if (warp == 0) {
    if (lane == 0) {
      int ait = 0, as = 0, bs = 0;
      uint32_t aph = 0, bph = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const int tm = tile % tiles_m, tn = tile / tiles_m;
        const int m0 = tm * BM;
        for (int cb = 0; cb < cblocks; ++cb, ++ait) {
          mbar_wait_sleep(&a_empty[as], aph ^ 1);
          if (ep.prof && blockIdx.x == 0 && cb == 0 && ait / cblocks < 16)
            ep.prof[4096 + (ait / cblocks) * 8 + 0] = clock64();
          uint8_t* sa = a_base + as * sh.a_stage_bytes;
          if constexpr (CH == 16) {
            // the 16-channel input is stored pre-swizzled (gg_stem_gather / gg_nchw_to_s2d16,
            // padded): one linear bulk copy of the span reproduces the SW32 image
            // (rows past the buffer end only feed discarded outputs)
            const int64_t rows_left = (int64_t)sh.N * img - m0;
            const int rows = rows_left < sh.span_rows ? (int)rows_left : sh.span_rows;
            mbar_expect_tx(&a_full[as], rows * RB);
            bulk_load(sa, ep.x16 + (int64_t)m0 * CH, rows * RB, &a_full[as]);
          } else {
            mbar_expect_tx(&a_full[as], sh.boxes * sh.box_rows * RB);
            for (int bx = 0; bx < sh.boxes; ++bx)   // boxes of <= 256 rows (TMA limit)
              tma_load_2d(sa + bx * sh.box_rows * RB, &map_x, &a_full[as], cb * CH, m0 + bx * sh.box_rows);
          }
          if (++as == AST) {
            as = 0;
            aph ^= 1;
          }
          if (!sh.bres) {
            for (int tap = 0; tap < TAPS; ++tap) {
              mbar_wait_sleep(&b_empty[bs], bph ^ 1);
              mbar_expect_tx(&b_full[bs], B_BYTES);
              tma_load_2d(b_base + bs * B_BYTES, &map_w, &b_full[bs], (cb * TAPS + tap) * CH, tn * BN);
              if (++bs == BST) {
                bs = 0;
                bph ^= 1;
              }
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    {   // the whole warp runs the loop; MMA batches / commits go out from one elected lane
      constexpr uint32_t idesc = idesc_act_f32(128, BN);
      uint64_t tap_off[TAPS];   // row shift of tap (r, s) in 16-B descriptor units
#pragma unroll
      for (int tap = 0; tap < TAPS; ++tap)
        tap_off[tap] = (uint64_t)(((tap / RT) * sh.Wp + tap % RT) * (RB / 16));
      long long wt[3] = {0, 0, 0};   // GG_SPAN_PROF: cycles waiting on acc_empty / A / B
      const long long t_mma0 = clock64();
#define SPAN_WAIT(bar, par, slot)                              \
  do {                                                         \
    if (ep.prof) {                                             \
      const long long t_ = clock64();                          \
      mbar_wait(bar, par);                                     \
      wt[slot] += clock64() - t_;                              \
    } else {                                                   \
      mbar_wait(bar, par);                                     \
    }                                                          \
  } while (0)
      if (b_loaded) mbar_wait(bres_full, 0);   // also when the count leaves no tile: drain the TMA
      const uint64_t bres_desc = sdesc_sw(smem_u32(b_base), RB);
      const uint64_t a_desc0 = sdesc_sw(smem_u32(a_base), RB);
      const uint64_t a_stage_d = (uint64_t)(sh.a_stage_bytes >> 4);
      int as = 0, bs = 0, t = 0;   // ring positions advance incrementally (lean issue chain)
      uint32_t aph = 0, bph = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++t) {
        const int acc = t % NACC;
        SPAN_WAIT(&acc_empty[acc], ((t / NACC) & 1) ^ 1, 0);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * ACC_COLS;
        for (int cb = 0; cb < cblocks; ++cb) {
          SPAN_WAIT(&a_full[as], aph, 1);
          if (ep.prof && blockIdx.x == 0 && cb == 0 && t < 16 && lane == 0) ep.prof[4096 + t * 8 + 1] = clock64();
          tc_fence_after();
          const uint64_t ad = a_desc0 + (uint64_t)as * a_stage_d;
          const int as_now = as;
          if (++as == AST) {
            as = 0;
            aph ^= 1;
          }
          if (sh.bres) {
            const uint64_t bd = bres_desc + (uint64_t)(cb * TAPS * (B_BYTES >> 4));
            if (elect_one_sync()) {
#pragma unroll
              for (int tap = 0; tap < TAPS; ++tap) {
                const uint64_t ao = ad + tap_off[tap];
                const uint64_t bo = bd + (uint64_t)(tap * (B_BYTES >> 4));
#pragma unroll
                for (int kk = 0; kk < KSTEPS; ++kk)
#pragma unroll
                  for (int mt = 0; mt < MT; ++mt)
                    umma_bf16(d_tmem + mt * BN, ao + (uint64_t)(mt * 128 * RB / 16 + kk * 2),
                              bo + (uint64_t)(kk * 2), idesc, (cb | tap | kk) != 0);
              }
              umma_commit(&a_empty[as_now]);
            }
            __syncwarp();
          } else {
#pragma unroll
            for (int tap = 0; tap < TAPS; ++tap) {
              SPAN_WAIT(&b_full[bs], bph, 2);
              tc_fence_after();
              const uint64_t ao = ad + tap_off[tap];
              const uint64_t bo = bres_desc + (uint64_t)bs * (uint64_t)(B_BYTES >> 4);
              if (elect_one_sync()) {
#pragma unroll
                for (int kk = 0; kk < KSTEPS; ++kk)
#pragma unroll
                  for (int mt = 0; mt < MT; ++mt)
                    umma_bf16(d_tmem + mt * BN, ao + (uint64_t)(mt * 128 * RB / 16 + kk * 2),
                              bo + (uint64_t)(kk * 2), idesc, (cb | tap | kk) != 0);
                umma_commit(&b_empty[bs]);
                if (tap == TAPS - 1) umma_commit(&a_empty[as_now]);
              }
              __syncwarp();
              if (++bs == BST) {
                bs = 0;
                bph ^= 1;
              }
            }
          }
        }
        if (elect_one_sync()) umma_commit(&acc_full[acc]);
        __syncwarp();
        if (ep.prof && blockIdx.x == 0 && t < 16 && lane == 0) ep.prof[4096 + t * 8 + 2] = clock64();
      }
#undef SPAN_WAIT
      if (ep.prof && lane == 0) {
        ep.prof[6144 + blockIdx.x * 4 + 0] = wt[0];
        ep.prof[6144 + blockIdx.x * 4 + 1] = wt[1];
        ep.prof[6144 + blockIdx.x * 4 + 2] = wt[2];
        ep.prof[6144 + blockIdx.x * 4 + 3] = clock64() - t_mma0;
      }
    }
  } else {
    // epilogue: warp w handles TMEM lane quarter (w % 4) and column half (w - 2) / 4
    const int quarter = warp & 3;
    const int half = (warp - 2) >> 2;
    constexpr int HALF = BN / 2;
    int t = 0;
    if (!DENSE && ep.tma_out) {
      // Coalesced epilogue (see conv_span_pair): 32 consecutive rows of a warp are 32
      // consecutive padded output rows -> one TMA box per 32 x 32 chunk, through a
      // per-warp SW64 staging buffer; the residual box comes in by TMA first.
      uint8_t* stg = stg_base + (warp - 2) * 4096;
      uint64_t* rb = res_full + (warp - 2) * 2;
      uint32_t rph[2] = {0, 0};
      const bool has_res = ep.residual != nullptr;
      const int sw = (lane >> 1) & 3;
      constexpr int NCH = HALF / 32;
      int gc = 0;   // running chunk counter: staging buffer gc & 1
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++t) {
        const int tm = tile % tiles_m, tn = tile / tiles_m;
        const int acc = t % NACC;
        const uint32_t tbase = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * ACC_COLS;
#pragma unroll 1
        for (int mt = 0; mt < MT; ++mt) {
          const int mw = tm * BM + mt * 128 + quarter * 32;
          const int orow0 = mw + sh.Wp + 1;
          const int colw = tn * BN + half * HALF;
          const bool any = mw < Mtot;
          const int m = mw + lane;
          const int nimg = m / img;
          const int within = m - nimg * img;
          const int h = within / sh.Wp, w = within - (within / sh.Wp) * sh.Wp;
          const bool real = m < Mtot && h < sh.Ho && w < sh.Wo;
#pragma unroll 1
          for (int c = 0; c < NCH; ++c, ++gc) {
            const int bsel = gc & 1;
            uint8_t* buf = stg + bsel * 2048;
            if (any && lane == 0) {
              bulk_wait_read<0>();   // earlier stores have read the staging buffers
              if (has_res) {
                mbar_expect_tx(&rb[bsel], 2048);
                tma_load_2d(buf, &map_res, &rb[bsel], colw + 32 * c, orow0);
              }
            }
            __syncwarp();
            if (mt == 0 && c == 0) {
              mbar_wait_sleep(&acc_full[acc], (t / NACC) & 1);
              tc_fence_after();
            }
            uint32_t r[32];
            tmem_ld_32x32b_x32(tbase + mt * BN + half * HALF + 32 * c, r);
            tmem_ld_wait();
            if (!any) continue;
            const int col0 = colw + 32 * c;
            uint4* myrow = reinterpret_cast<uint4*>(buf + lane * 64);
            float v[32];
            if (has_res) {
              mbar_wait(&rb[bsel], rph[bsel]);
              rph[bsel] ^= 1;
            }
            if (real) {
#pragma unroll
              for (int i = 0; i < 32; i += 4) {
                const float4 bb = __ldg(reinterpret_cast<const float4*>(ep.bias + col0 + i));
                v[i] = __uint_as_float(r[i]) + bb.x;
                v[i + 1] = __uint_as_float(r[i + 1]) + bb.y;
                v[i + 2] = __uint_as_float(r[i + 2]) + bb.z;
                v[i + 3] = __uint_as_float(r[i + 3]) + bb.w;
              }
              if (has_res) {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                  const uint4 u = myrow[q ^ sw];
                  const act2_t* h2 = reinterpret_cast<const act2_t*>(&u);
#pragma unroll
                  for (int e = 0; e < 4; ++e) {
                    const float2 f = act2_to_float2(h2[e]);
                    v[q * 8 + 2 * e] += f.x;
                    v[q * 8 + 2 * e + 1] += f.y;
                  }
                }
              }
              if (ep.relu) {
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] = fmaxf(v[i], 0.0f);
              }
            } else {
#pragma unroll
              for (int i = 0; i < 32; ++i) v[i] = 0.0f;
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              uint4 u;
              u.x = pack_act(v[q * 8 + 0], v[q * 8 + 1]);
              u.y = pack_act(v[q * 8 + 2], v[q * 8 + 3]);
              u.z = pack_act(v[q * 8 + 4], v[q * 8 + 5]);
              u.w = pack_act(v[q * 8 + 6], v[q * 8 + 7]);
              myrow[q ^ sw] = u;
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store_2d(&map_out, buf, col0, orow0);
              bulk_commit();
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[acc]);
      }
      if (lane == 0) bulk_wait<0>();
    }
    if (DENSE || !ep.tma_out)
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++t) {
      const int tm = tile % tiles_m, tn = tile / tiles_m;
      const int acc = t % NACC;
      mbar_wait_sleep(&acc_full[acc], (t / NACC) & 1);
      if (ep.prof && blockIdx.x == 0 && warp == 2 && lane == 0 && t < 16) ep.prof[4096 + t * 8 + 3] = clock64();
      tc_fence_after();
#pragma unroll 1
      for (int mt = 0; mt < (ep.nostore == 2 ? 0 : MT); ++mt) {   // nostore 2: skip the epilogue (debug)
        const int m = tm * BM + mt * 128 + quarter * 32 + lane;
        const int nimg = m / img;
        const int within = m - nimg * img;
        const int h = within / sh.Wp, w = within - (within / sh.Wp) * sh.Wp;
        const bool real = m < Mtot && h < sh.Ho && w < sh.Wo;
        int64_t oidx;
        bool store;
        if constexpr (DENSE) {
          oidx = ((int64_t)nimg * sh.Ho + h) * sh.Wo + w;
          store = real;
        } else {
          oidx = (int64_t)m + sh.Wp + 1;   // padded output position
          store = m < Mtot && oidx < (int64_t)n_eff * img;
        }
        const uint32_t tcol = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * ACC_COLS + mt * BN;
#pragma unroll 1
        for (int c = half * HALF; c < (half + 1) * HALF; c += 32) {
          const int col0 = tn * BN + c;
          // residual loads first: their latency overlaps the TMEM read
          uint4 res[4];
          const bool use_res = !DENSE && ep.residual != nullptr && store && real;
          if (use_res) {
            const uint4* rp = reinterpret_cast<const uint4*>(ep.residual + oidx * sh.Cout + col0);
#pragma unroll
            for (int q = 0; q < 4; ++q) res[q] = __ldg(rp + q);
          }
          uint32_t r[32];
          tmem_ld_32x32b_x32(tcol + c, r);
          tmem_ld_wait();
          if (DENSE && !ep.nostore) {
            // stem (dense output rows): coalesced stores through the warp's smem tile
            float v[32];
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
              const float4 b = __ldg(reinterpret_cast<const float4*>(ep.bias + col0 + i));
              v[i] = __uint_as_float(r[i]) + b.x;
              v[i + 1] = __uint_as_float(r[i + 1]) + b.y;
              v[i + 2] = __uint_as_float(r[i + 2]) + b.z;
              v[i + 3] = __uint_as_float(r[i + 3]) + b.w;
            }
            if (ep.relu) {
#pragma unroll
              for (int i = 0; i < 32; ++i) v[i] = fmaxf(v[i], 0.0f);
            }
            uint4 outr[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              outr[q].x = pack_act(v[q * 8 + 0], v[q * 8 + 1]);
              outr[q].y = pack_act(v[q * 8 + 2], v[q * 8 + 3]);
              outr[q].z = pack_act(v[q * 8 + 4], v[q * 8 + 5]);
              outr[q].w = pack_act(v[q * 8 + 6], v[q * 8 + 7]);
            }
            // the stem output (103 MB at batch 64) is read once by the max pool right
            // after: keep it in L2 (evict_last); the pool reads it evict_first
            warp_rows_store<true>(stg_base + (warp - 2) * 4096, ep.y, oidx * sh.Cout + col0, store, lane, outr);
            continue;
          }
          if (!store) continue;
          float v[32];
          if (real) {
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
              const float4 b = __ldg(reinterpret_cast<const float4*>(ep.bias + col0 + i));
              v[i] = __uint_as_float(r[i]) + b.x;
              v[i + 1] = __uint_as_float(r[i + 1]) + b.y;
              v[i + 2] = __uint_as_float(r[i + 2]) + b.z;
              v[i + 3] = __uint_as_float(r[i + 3]) + b.w;
            }
            if (use_res) {
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const act2_t* h2 = reinterpret_cast<const act2_t*>(&res[q]);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const float2 f = act2_to_float2(h2[e]);
                  v[q * 8 + 2 * e] += f.x;
                  v[q * 8 + 2 * e + 1] += f.y;
                }
              }
            }
            if (ep.relu) {
#pragma unroll
              for (int i = 0; i < 32; ++i) v[i] = fmaxf(v[i], 0.0f);
            }
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = 0.0f;   // padding positions stay zero
          }
          if (ep.nostore) continue;
          uint4* dp = reinterpret_cast<uint4*>(ep.y + oidx * sh.Cout + col0);
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
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[acc]);
      if (ep.prof && blockIdx.x == 0 && warp == 2 && lane == 0 && t < 16) ep.prof[4096 + t * 8 + 4] = clock64();
    }
  }
  __syncthreads();
  if (ep.prof && threadIdx.x == 0) {
    ep.prof[2 * blockIdx.x + 1] = gtimer();
    ep.prof[2048 + 2 * blockIdx.x + 1] = clock64();
  }
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, NACC * ACC_COLS);
  }
}

// 2-D map over a [rows, cols] bf16 matrix, box [ch, box_rows], swizzle by row bytes.
static int make_map_span(CUtensorMap* map, const void* ptr, int64_t rows, int64_t cols, int ch,
                         int box_rows, bool preswizzled = false) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  if (!enc) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return GG_ERR_CUDA;
    enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {(cuuint32_t)ch, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(ptr), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   preswizzled ? CU_TENSOR_MAP_SWIZZLE_NONE
                   : ch == 64  ? CU_TENSOR_MAP_SWIZZLE_128B
                               : CU_TENSOR_MAP_SWIZZLE_32B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? GG_OK : GG_ERR_INVALID_ARGUMENT;
}

// [rows, cols] bf16 (row pitch = cols), box 32 x 32, 64-byte swizzle: the pair
// conv's TMA epilogue boxes (outputs and residuals in the padded geometry).
static int make_map_box32(CUtensorMap* map, const void* ptr, int64_t rows, int64_t cols) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  if (!enc) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return GG_ERR_CUDA;
    enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(ptr), dims, strides, box,
                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? GG_OK : GG_ERR_INVALID_ARGUMENT;
}

static int span_smem_bytes(const SpanShape& sh, int bn, int rb, int taps) {
  const int nkb = sh.C / (rb / 2) * taps;
  return sh.a_stages * sh.a_stage_bytes + (sh.bres ? nkb : sh.b_stages) * bn * rb + 1024 + 1024;
}

template <int BN, int CH, int RT, bool DENSE, int MT>
static int launch_span(const CUtensorMap& mx, const CUtensorMap& mw, const SpanShape& sh,
                       const SpanEpi& ep, cudaStream_t s, const CUtensorMap* mo = nullptr,
                       const CUtensorMap* mr = nullptr) {
  auto kern = conv_span_tcgen05<BN, CH, RT, DENSE, MT>;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSpanSmemMax) != cudaSuccess)
      return GG_ERR_CUDA;
    attr = true;
  }
  const int smem = span_smem_bytes(sh, BN, CH * 2, RT * RT) + ((ep.tma_out || DENSE) ? kSpanStgBytes : 0);
  const int tiles = ((sh.N * sh.Hp * sh.Wp + 128 * MT - 1) / (128 * MT)) * (sh.Cout / BN);
  const int grid = tiles < num_sms() ? tiles : num_sms();
  SpanEpi e2 = ep;
  e2.nostore = getenv("GG_SPAN_NOSTORE") ? atoi(getenv("GG_SPAN_NOSTORE")) : 0;
  static unsigned long long* prof = nullptr;
  const bool do_prof = getenv("GG_SPAN_PROF") != nullptr;
  if (do_prof) {
    if (!prof) cudaMalloc(&prof, 8 * 1024 * sizeof(unsigned long long));
    e2.prof = prof;
    cudaMemsetAsync(prof + 4096, 0, 4096 * sizeof(unsigned long long), s);
  }
  static int prof_calls = 0;
  const int prof_at = do_prof ? atoi(getenv("GG_SPAN_PROF")) : 0;
  const bool report = do_prof && ++prof_calls >= (prof_at > 0 ? prof_at : 1);
  if (launch_pdl(kern, dim3(grid), dim3(kSpanThreads), smem, s, mx, mw, mo ? *mo : mx, mr ? *mr : mx, sh,
                 e2) != cudaSuccess)
    return GG_ERR_CUDA;
  if (report) {
    prof_calls = 0;
    static unsigned long long h[8 * 1024];
    cudaDeviceSynchronize();
    cudaMemcpy(h, prof, 8 * 1024 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    const unsigned long long c0 = h[2048];
    fprintf(stderr, "CTA0 timeline (cycles from CTA start): tile: tma_issue a_full mma_issued epi_got epi_done\n");
    for (int t = 0; t < 16; ++t) {
      const unsigned long long* e = h + 4096 + t * 8;
      if (!e[1]) break;
      fprintf(stderr, "  %2d: %7lld %7lld %7lld %7lld %7lld\n", t, (long long)(e[0] - c0),
              (long long)(e[1] - c0), (long long)(e[2] - c0), (long long)(e[3] - c0), (long long)(e[4] - c0));
    }
    double csum = 0;
    for (int i = 0; i < grid; ++i) csum += (double)(h[2048 + 2 * i + 1] - h[2048 + 2 * i]);
    fprintf(stderr, "span mean CTA clock64 cycles %.0f\n", csum / grid);
    double w0 = 0, w1 = 0, w2 = 0, wt = 0;
    for (int i = 0; i < grid; ++i) {
      w0 += (double)h[6144 + 4 * i];
      w1 += (double)h[6144 + 4 * i + 1];
      w2 += (double)h[6144 + 4 * i + 2];
      wt += (double)h[6144 + 4 * i + 3];
    }
    fprintf(stderr, "MMA issuer (mean over CTAs): %.0f cycles, waiting acc_empty %.0f%%, A %.0f%%, B %.0f%%\n",
            wt / grid, 100 * w0 / wt, 100 * w1 / wt, 100 * w2 / wt);
    unsigned long long s0 = ~0ull, s1 = 0, e0 = ~0ull, e1 = 0;
    double dsum = 0;
    for (int i = 0; i < grid; ++i) {
      s0 = h[2 * i] < s0 ? h[2 * i] : s0;
      s1 = h[2 * i] > s1 ? h[2 * i] : s1;
      e0 = h[2 * i + 1] < e0 ? h[2 * i + 1] : e0;
      e1 = h[2 * i + 1] > e1 ? h[2 * i + 1] : e1;
      dsum += (double)(h[2 * i + 1] - h[2 * i]);
    }
    fprintf(stderr, "span BN=%d CH=%d RT=%d MT=%d C=%d Cout=%d H=%d: grid %d tiles %d stages A%d B%d%s | "
            "start spread %.2f us, end spread %.2f us, mean CTA %.2f us, total %.2f us\n",
            BN, CH, RT, MT, sh.C, sh.Cout, sh.H, grid, tiles, sh.a_stages, sh.b_stages,
            sh.bres ? " (B resident)" : "", (s1 - s0) * 1e-3, (e1 - e0) * 1e-3, dsum / grid * 1e-3,
            (e1 - s0) * 1e-3);
  }
  return GG_OK;
}


// ---------------------------------------------------------------------------
// CTA-pair span convolution (cluster of 2, cta_group::2) for the 3x3/1 convs of
// layers 2-4.  Why: a cta_group::1 128 x N x 16 MMA reads (4 KB + N * 32 B) of
// shared memory per N/2 cycles — at N = 128 that is the SM's whole 128 B/cycle
// of smem bandwidth, so the TMA writes of the operand ring push the tensor pipe
// to ~80 cycles per 64-cycle MMA (measured with GG_SPAN_PROF: the issuer waits
// on loads only ~15 % of the time).  A pair MMA (M = 256 over two SMs, each CTA
// holding its own 128 rows of A and half of the N columns of B) reads 64 B/cycle
// per SM at N = 256 (96 at N = 128), and each SM streams only half of the
// weight slabs.
// Tile of the pair: output rows [tm*256, tm*256+256) of the padded space (CTA
// rank r owns 128 of them, with its own A span) x BN output channels.
template <int BN, int CH, int RT, bool DENSE>
__global__ void __launch_bounds__(kSpanThreads, 1)
    conv_span_pair(const __grid_constant__ CUtensorMap map_x, const __grid_constant__ CUtensorMap map_w,
                   const __grid_constant__ CUtensorMap map_out, const __grid_constant__ CUtensorMap map_res,
                   SpanShape sh, SpanEpi ep) {
  constexpr int RB = CH * 2;                 // bytes per pixel row
  constexpr int KSTEPS = CH / 16;            // MMAs per tap
  constexpr int TAPS = RT * RT;
  constexpr int BH = BN / 2;                 // B rows per CTA (its half of the N tile)
  constexpr int B_BYTES = BH * RB;           // one tap slab of this CTA's B half
  constexpr int NACC = 512 / BN >= 4 ? 4 : 2;   // TMEM accumulator buffers
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_align1k(smem_raw);
  const int cblocks = sh.C / CH;
  const int nkb = cblocks * TAPS;
  const int AST = sh.a_stages, BST = sh.b_stages;
  uint8_t* a_base = smem;
  uint8_t* b_base = smem + AST * sh.a_stage_bytes;
  const int b_slots = sh.bres ? nkb : BST;
  uint64_t* bars = reinterpret_cast<uint64_t*>(b_base + b_slots * B_BYTES);
  uint64_t* a_full = bars;
  uint64_t* a_empty = a_full + kSpanMaxStages;
  uint64_t* b_full = a_empty + kSpanMaxStages;
  uint64_t* b_empty = b_full + kSpanMaxStages;
  uint64_t* acc_full = b_empty + kSpanMaxStages;
  uint64_t* acc_empty = acc_full + NACC;
  uint64_t* bres_full = acc_empty + NACC;
  uint64_t* res_full = bres_full + 1;      // [8 warps][2]: residual boxes landed (TMA epilogue)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(res_full + 2 * kSpanEpiWarps);
  // TMA epilogue staging: per epilogue warp two 2 KB SW64 images of 32 x 32 bf16 boxes
  uint8_t* stg_base = smem_align1k(reinterpret_cast<uint8_t*>(bars) + 1024);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  griddep_launch();
  const int img = sh.Hp * sh.Wp;
  const int tiles_n = sh.Cout / BN;

  if (threadIdx.x == 0) {
    for (int i = 0; i < AST; ++i) {   // only the ring slots this launch uses
      mbar_init(&a_full[i], 1);
      mbar_init(&a_empty[i], 1);
    }
    for (int i = 0; i < BST; ++i) {
      mbar_init(&b_full[i], 1);
      mbar_init(&b_empty[i], 1);
    }
    for (int i = 0; i < NACC; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 2 * kSpanEpiWarps);
    }
    mbar_init(bres_full, 1);
    for (int i = 0; i < 2 * kSpanEpiWarps; ++i) mbar_init(&res_full[i], 1);
    fence_mbar_init();
    tma_prefetch(&map_x);
    tma_prefetch(&map_w);
    if (ep.tma_out) {
      tma_prefetch(&map_out);
      if (ep.residual) tma_prefetch(&map_res);
    }
  }
  if (warp == 1) tmem_alloc_pair(tmem_slot, NACC * BN);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // resident weights (this CTA's half of the single N tile): independent of the predecessor
  const int tiles_max = (sh.N * img + 255) / 256 * tiles_n;
  const bool b_loaded = sh.bres && tiles_max > pair;
  if (warp == 0 && lane == 0 && b_loaded) {
    const uint32_t fb = mapa_shared(smem_u32(bres_full), 0);
    if (rank == 0) mbar_expect_tx(bres_full, 2 * nkb * B_BYTES);
    for (int kb = 0; kb < nkb; ++kb)
      tma_load_2d_pair(b_base + kb * B_BYTES, &map_w, fb, kb * CH, rank * BH);
  }
  griddep_wait();
  const int n_eff = ep.count ? min(sh.N, __ldg(ep.count)) : sh.N;
  const int Mtot = n_eff * img;
  const int tiles_m = (Mtot + 255) / 256;
  const int num_tiles = tiles_m * tiles_n;

  if (warp == 0) {
    if (lane == 0) {
      // ring positions advance incrementally (no runtime % and / per load)
      int as = 0, bs = 0;
      uint32_t aph = 0, bph = 0;
      SkSched sc(ep.sk.enabled, num_tiles, cblocks, pair, npairs);
      SkWork wk;
      while (sc.next(wk)) {
        const int tile = wk.tile;
        const int tm = tile % tiles_m, tn = tile / tiles_m;
        const int m0 = tm * 256 + rank * 128;
        for (int cb = wk.kb0; cb < wk.kb1; ++cb) {
          mbar_wait_sleep(&a_empty[as], aph ^ 1);
          uint8_t* sa = a_base + as * sh.a_stage_bytes;
          const uint32_t fa = mapa_shared(smem_u32(&a_full[as]), 0);
          if (rank == 0) mbar_expect_tx(&a_full[as], 2 * sh.boxes * sh.box_rows * RB);
          for (int bx = 0; bx < sh.boxes; ++bx)
            tma_load_2d_pair(sa + bx * sh.box_rows * RB, &map_x, fa, cb * CH, m0 + bx * sh.box_rows);
          if (++as == AST) {
            as = 0;
            aph ^= 1;
          }
          if (!sh.bres) {
            for (int tap = 0; tap < TAPS; ++tap) {
              mbar_wait_sleep(&b_empty[bs], bph ^ 1);
              const uint32_t fb = mapa_shared(smem_u32(&b_full[bs]), 0);
              if (rank == 0) mbar_expect_tx(&b_full[bs], 2 * B_BYTES);
              tma_load_2d_pair(b_base + bs * B_BYTES, &map_w, fb, (cb * TAPS + tap) * CH,
                               tn * BN + rank * BH);
              if (++bs == BST) {
                bs = 0;
                bph ^= 1;
              }
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {   // leader: the warp runs the loop, one elected lane issues
      constexpr uint32_t idesc = idesc_act_f32(256, BN);
      uint64_t tap_off[TAPS];
#pragma unroll
      for (int tap = 0; tap < TAPS; ++tap) tap_off[tap] = (uint64_t)(((tap / RT) * sh.Wp + tap % RT) * (RB / 16));
      if (b_loaded) mbar_wait(bres_full, 0);
      const uint64_t bres_desc = sdesc_sw(smem_u32(b_base), RB);
      const uint64_t a_desc0 = sdesc_sw(smem_u32(a_base), RB);
      const uint64_t a_stage_d = (uint64_t)(sh.a_stage_bytes >> 4);
      // one dependent instruction stream feeds the tensor pipe: ring positions and
      // descriptors advance incrementally (no runtime % and / per tap)
      int as = 0, bs = 0, t = 0;
      uint32_t aph = 0, bph = 0;
      long long wt_acc = 0, wt_a = 0, wt_b = 0;   // GG_SPAN_PROF: issuer wait cycles
      const long long t_mma0 = clock64();
#define GG_PAIR_WAIT(bar, par, acc_)                    \
  do {                                                  \
    if (ep.prof) {                                      \
      const long long t_ = clock64();                   \
      mbar_wait(bar, par);                              \
      acc_ += clock64() - t_;                           \
    } else {                                            \
      mbar_wait(bar, par);                              \
    }                                                   \
  } while (0)
      SkSched sc(ep.sk.enabled, num_tiles, cblocks, pair, npairs);
      SkWork wk;
      for (; sc.next(wk); ++t) {
        const int acc = t % NACC;
        GG_PAIR_WAIT(&acc_empty[acc], ((t / NACC) & 1) ^ 1, wt_acc);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int cb = wk.kb0; cb < wk.kb1; ++cb) {
          GG_PAIR_WAIT(&a_full[as], aph, wt_a);
          tc_fence_after();
          const uint64_t ad = a_desc0 + (uint64_t)as * a_stage_d;
          const int as_now = as;
          if (++as == AST) {
            as = 0;
            aph ^= 1;
          }
          if (sh.bres) {
            const uint64_t bd = bres_desc + (uint64_t)(cb * TAPS * (B_BYTES >> 4));
            if (elect_one_sync()) {
#pragma unroll
              for (int tap = 0; tap < TAPS; ++tap) {
                const uint64_t ao = ad + tap_off[tap];
                const uint64_t bo = bd + (uint64_t)(tap * (B_BYTES >> 4));
#pragma unroll
                for (int kk = 0; kk < KSTEPS; ++kk)
                  umma_bf16_pair(d_tmem, ao + (uint64_t)(kk * 2), bo + (uint64_t)(kk * 2), idesc,
                                 (cb != wk.kb0 || tap != 0 || kk != 0));
              }
              umma_commit_pair(&a_empty[as_now], 3);
            }
            __syncwarp();
          } else {
#pragma unroll
            for (int tap = 0; tap < TAPS; ++tap) {
              GG_PAIR_WAIT(&b_full[bs], bph, wt_b);
              tc_fence_after();
              const uint64_t ao = ad + tap_off[tap];
              const uint64_t bo = bres_desc + (uint64_t)bs * (uint64_t)(B_BYTES >> 4);
              if (elect_one_sync()) {
#pragma unroll
                for (int kk = 0; kk < KSTEPS; ++kk)
                  umma_bf16_pair(d_tmem, ao + (uint64_t)(kk * 2), bo + (uint64_t)(kk * 2), idesc,
                                 (cb != wk.kb0 || tap != 0 || kk != 0));
                umma_commit_pair(&b_empty[bs], 3);
                if (tap == TAPS - 1) umma_commit_pair(&a_empty[as_now], 3);
              }
              __syncwarp();
              if (++bs == BST) {
                bs = 0;
                bph ^= 1;
              }
            }
          }
        }
        if (elect_one_sync()) umma_commit_pair(&acc_full[acc], 3);
        __syncwarp();
      }
#undef GG_PAIR_WAIT
      if (ep.prof && lane == 0) {
        ep.prof[6144 + pair * 4 + 0] = wt_acc;
        ep.prof[6144 + pair * 4 + 1] = wt_a;
        ep.prof[6144 + pair * 4 + 2] = wt_b;
        ep.prof[6144 + pair * 4 + 3] = clock64() - t_mma0;
        ep.prof[4096 + pair] = t;
      }
    }
  } else {
    const int quarter = warp & 3;
    const int half = (warp - 2) >> 2;
    constexpr int HALF = BN / 2;
    const uint32_t leader_empty0 = mapa_shared(smem_u32(&acc_empty[0]), 0);
    int t = 0;
    if (!DENSE && ep.tma_out) {
      // Coalesced epilogue (as in gemm_bf16_pair): the warp's 32 consecutive rows m
      // map to 32 consecutive padded output rows m + Wp + 1, so each 32 x 32 chunk
      // is one TMA box; rows that are padding (or past the batch) are written as 0.
      uint8_t* stg = stg_base + (warp - 2) * 4096;
      uint64_t* rb = res_full + (warp - 2) * 2;
      uint32_t rph0 = 0, rph1 = 0;
      const bool has_res = ep.residual != nullptr;
      const int sw = (lane >> 1) & 3;
      constexpr int NCH = HALF / 32;   // chunks per warp
      SkSched sc(ep.sk.enabled, num_tiles, cblocks, pair, npairs);
      SkWork wk;
      for (; sc.next(wk); ++t) {
        const int tile = wk.tile;
        const int tm = tile % tiles_m, tn = tile / tiles_m;
        const int acc = t % NACC;
        // stream-K: a tile cut between pairs is reduced by its last arriving segment;
        // each (rank, epilogue warp) region of 32 rows x HALF columns has its own
        // arrival / ready counters and fp32 partial slots (column-major: coalesced)
        const bool partial = wk.kb0 != 0 || wk.kb1 != cblocks;
        const int region = (int)rank * kSpanEpiWarps + (warp - 2);
        constexpr int kRegions = 2 * kSpanEpiWarps;
        int c_first = 0, c_last = 0;
        if (partial) {
          c_first = sc.cta_of((int64_t)tile * cblocks);
          c_last = sc.cta_of((int64_t)tile * cblocks + cblocks - 1);
          const int nseg = c_last - c_first + 1;
          int* cnt = ep.sk.cnt + ((int64_t)tile * kRegions + region) * 2;
          mbar_wait_sleep(&acc_full[acc], (t / NACC) & 1);
          tc_fence_after();
          int arrive = 0;
          if (lane == 0) arrive = atomicAdd(cnt, 1);
          arrive = __shfl_sync(0xffffffffu, arrive, 0);
          if (arrive < nseg - 1) {   // write this segment's partial and leave
            const int slot = (tile == (int)(sc.start_of(pair) / cblocks)) ? 0 : 1;
            float* dst = ep.sk.ws + (((int64_t)pair * 2 + slot) * kRegions + region) * (32 * HALF);
            const uint32_t tb = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * BN + half * HALF;
#pragma unroll 1
            for (int c = 0; c < NCH; ++c) {
              uint32_t r[32];
              tmem_ld_32x32b_x32(tb + 32 * c, r);
              tmem_ld_wait();
#pragma unroll
              for (int i = 0; i < 32; ++i) __stcg(dst + (32 * c + i) * 32 + lane, __uint_as_float(r[i]));
            }
            __threadfence();
            __syncwarp();
            if (lane == 0) atomicAdd(cnt + 1, 1);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(leader_empty0 + acc * 8);
            continue;
          }
          while (ld_acquire(cnt + 1) < nseg - 1) __nanosleep(64);
          __syncwarp();
          if (lane == 0) {   // reset for the next launch (stream-ordered)
            cnt[0] = 0;
            cnt[1] = 0;
          }
        }
        const int mw = tm * 256 + rank * 128 + quarter * 32;   // the warp's first row
        const int orow0 = mw + sh.Wp + 1;
        const int colw = tn * BN + half * HALF;
        const bool any = mw < Mtot;
        if (has_res && any && lane == 0) {
          bulk_wait_read<0>();
          mbar_expect_tx(&rb[0], 2048);
          tma_load_2d(stg, &map_res, &rb[0], colw, orow0);
        }
        if (!partial) {
          mbar_wait_sleep(&acc_full[acc], (t / NACC) & 1);
          tc_fence_after();
        }
        const int m = mw + lane;
        const int nimg = m / img;
        const int within = m - nimg * img;
        const int h = within / sh.Wp, w = within - (within / sh.Wp) * sh.Wp;
        const bool real = m < Mtot && h < sh.Ho && w < sh.Wo;
        const uint32_t tcol = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * BN + half * HALF;
#pragma unroll 1
        for (int c = 0; c < NCH; ++c) {
          const int bsel = c & 1;
          uint8_t* buf = stg + bsel * 2048;
          if (any && lane == 0) {
            if (has_res) {
              if (c + 1 < NCH) {
                bulk_wait_read<0>();
                mbar_expect_tx(&rb[bsel ^ 1], 2048);
                tma_load_2d(stg + (bsel ^ 1) * 2048, &map_res, &rb[bsel ^ 1], colw + 32 * (c + 1), orow0);
              }
            } else {
              bulk_wait_read<1>();
            }
          }
          __syncwarp();
          uint32_t r[32];
          tmem_ld_32x32b_x32(tcol + 32 * c, r);
          tmem_ld_wait();
          if (partial) {   // k-ordered sum of the tile's segments (deterministic)
            float accv[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) accv[i] = 0.0f;
#pragma unroll 1
            for (int seg = c_first; seg <= c_last; ++seg) {
              if (seg == pair) {
#pragma unroll
                for (int i = 0; i < 32; ++i) accv[i] += __uint_as_float(r[i]);
              } else {
                const int slot = (tile == (int)(sc.start_of(seg) / cblocks)) ? 0 : 1;
                const float* src = ep.sk.ws + (((int64_t)seg * 2 + slot) * kRegions + region) * (32 * HALF);
                float pv[32];
#pragma unroll
                for (int i = 0; i < 32; ++i) pv[i] = __ldcg(src + (32 * c + i) * 32 + lane);
#pragma unroll
                for (int i = 0; i < 32; ++i) accv[i] += pv[i];
              }
            }
#pragma unroll
            for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(accv[i]);
          }
          if (!any) continue;
          const int col0 = colw + 32 * c;
          uint4* myrow = reinterpret_cast<uint4*>(buf + lane * 64);
          float v[32];
          if (has_res) {
            if (bsel == 0) { mbar_wait(&rb[0], rph0); rph0 ^= 1; }
            else { mbar_wait(&rb[1], rph1); rph1 ^= 1; }
          }
          if (real) {
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
              const float4 bb = __ldg(reinterpret_cast<const float4*>(ep.bias + col0 + i));
              v[i] = __uint_as_float(r[i]) + bb.x;
              v[i + 1] = __uint_as_float(r[i + 1]) + bb.y;
              v[i + 2] = __uint_as_float(r[i + 2]) + bb.z;
              v[i + 3] = __uint_as_float(r[i + 3]) + bb.w;
            }
            if (has_res) {
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const uint4 u = myrow[q ^ sw];
                const act2_t* h2 = reinterpret_cast<const act2_t*>(&u);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const float2 f = act2_to_float2(h2[e]);
                  v[q * 8 + 2 * e] += f.x;
                  v[q * 8 + 2 * e + 1] += f.y;
                }
              }
            }
            if (ep.relu) {
#pragma unroll
              for (int i = 0; i < 32; ++i) v[i] = fmaxf(v[i], 0.0f);
            }
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = 0.0f;   // padding positions / past the batch
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint4 u;
            u.x = pack_act(v[q * 8 + 0], v[q * 8 + 1]);
            u.y = pack_act(v[q * 8 + 2], v[q * 8 + 3]);
            u.z = pack_act(v[q * 8 + 4], v[q * 8 + 5]);
            u.w = pack_act(v[q * 8 + 6], v[q * 8 + 7]);
            myrow[q ^ sw] = u;
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&map_out, buf, col0, orow0);
            bulk_commit();
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(leader_empty0 + acc * 8);
      }
      if (lane == 0) bulk_wait<0>();
    }
    if (DENSE || !ep.tma_out)
    for (int tile = pair; tile < num_tiles; tile += npairs, ++t) {
      const int tm = tile % tiles_m, tn = tile / tiles_m;
      const int acc = t % NACC;
      mbar_wait_sleep(&acc_full[acc], (t / NACC) & 1);
      tc_fence_after();
      const int m = tm * 256 + rank * 128 + quarter * 32 + lane;
      const int nimg = m / img;
      const int within = m - nimg * img;
      const int h = within / sh.Wp, w = within - (within / sh.Wp) * sh.Wp;
      const bool real = m < Mtot && h < sh.Ho && w < sh.Wo;
      // padded mode: output at the padded position m + Wp + 1 (borders written as zeros);
      // dense mode (stem): real positions only, [N, Ho, Wo] layout
      const int64_t oidx = DENSE ? ((int64_t)nimg * sh.Ho + h) * sh.Wo + w : (int64_t)m + sh.Wp + 1;
      const bool store = DENSE ? real : (m < Mtot && oidx < (int64_t)n_eff * img);
      const uint32_t tcol = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * BN;
#pragma unroll 1
      for (int c = half * HALF; c < (half + 1) * HALF; c += 32) {
        const int col0 = tn * BN + c;
        uint4 res[4];
        const bool use_res = !DENSE && ep.residual != nullptr && store && real;
        if (use_res) {
          const uint4* rp = reinterpret_cast<const uint4*>(ep.residual + oidx * sh.Cout + col0);
#pragma unroll
          for (int q = 0; q < 4; ++q) res[q] = __ldg(rp + q);
        }
        uint32_t r[32];
        tmem_ld_32x32b_x32(tcol + c, r);
        tmem_ld_wait();
        if (!store) continue;
        float v[32];
        if (real) {
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            const float4 b = __ldg(reinterpret_cast<const float4*>(ep.bias + col0 + i));
            v[i] = __uint_as_float(r[i]) + b.x;
            v[i + 1] = __uint_as_float(r[i + 1]) + b.y;
            v[i + 2] = __uint_as_float(r[i + 2]) + b.z;
            v[i + 3] = __uint_as_float(r[i + 3]) + b.w;
          }
          if (use_res) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const act2_t* h2 = reinterpret_cast<const act2_t*>(&res[q]);
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float2 f = act2_to_float2(h2[e]);
                v[q * 8 + 2 * e] += f.x;
                v[q * 8 + 2 * e + 1] += f.y;
              }
            }
          }
          if (ep.relu) {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = fmaxf(v[i], 0.0f);
          }
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = 0.0f;   // padding positions stay zero
        }
        uint4* dp = reinterpret_cast<uint4*>(ep.y + oidx * sh.Cout + col0);
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
      if (lane == 0) mbar_arrive_cluster(leader_empty0 + acc * 8);
    }
  }
  __syncthreads();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, NACC * BN);
  }
}

template <int BN, int CH = 64, int RT = 3, bool DENSE = false>
static int launch_span_pair(const CUtensorMap& mx, const CUtensorMap& mw, const SpanShape& sh,
                            const SpanEpi& ep, cudaStream_t s, const CUtensorMap* mo = nullptr,
                            const CUtensorMap* mr = nullptr) {
  auto kern = conv_span_pair<BN, CH, RT, DENSE>;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSpanSmemMax) != cudaSuccess)
      return GG_ERR_CUDA;
    attr = true;
  }
  const int smem = span_smem_bytes(sh, BN / 2, CH * 2, RT * RT) + (ep.tma_out ? kSpanStgBytes : 0);
  const int tiles = ((sh.N * sh.Hp * sh.Wp + 255) / 256) * (sh.Cout / BN);
  const int pairs = num_sms() / 2;
  const int grid = ep.sk.enabled ? 2 * pairs : 2 * (tiles < pairs ? tiles : pairs);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kSpanThreads);
  cfg.dynamicSmemBytes = smem;
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
  static unsigned long long* prof = nullptr;
  SpanEpi e2 = ep;
  const bool do_prof = getenv("GG_SPAN_PROF") != nullptr;
  if (do_prof) {
    if (!prof) cudaMalloc(&prof, 8 * 1024 * sizeof(unsigned long long));
    cudaMemsetAsync(prof, 0, 8 * 1024 * sizeof(unsigned long long), s);
    e2.prof = prof;
  }
  if (cudaLaunchKernelEx(&cfg, kern, mx, mw, mo ? *mo : mx, mr ? *mr : mx, sh, e2) != cudaSuccess)
    return GG_ERR_CUDA;
  if (do_prof) {
    static unsigned long long h[8 * 1024];
    cudaDeviceSynchronize();
    cudaMemcpy(h, prof, sizeof(h), cudaMemcpyDeviceToHost);
    const int np = grid / 2;
    double w0 = 0, w1 = 0, w2 = 0, wt = 0, tl = 0, tmax = 0;
    for (int i = 0; i < np; ++i) {
      w0 += (double)h[6144 + 4 * i];
      w1 += (double)h[6144 + 4 * i + 1];
      w2 += (double)h[6144 + 4 * i + 2];
      wt += (double)h[6144 + 4 * i + 3];
      tl += (double)h[4096 + i];
      tmax = (double)h[4096 + i] > tmax ? (double)h[4096 + i] : tmax;
    }
    const double mma_cyc = (double)(sh.C / CH) * RT * RT * (CH / 16) * (BN >= 128 ? 64.0 * BN / 128 : 48.0);
    fprintf(stderr, "span pair BN=%d C=%d Cout=%d H=%d Wp=%d: %d pairs, tiles %.2f/pair (max %.0f), issuer %.0f cycles/pair, "
            "waiting acc %.0f%% A %.0f%% B %.0f%%, MMA-bound %.0f cycles/tile, stages A%d B%d%s\n",
            BN, sh.C, sh.Cout, sh.H, sh.Wp, np, tl / np, tmax, wt / np, 100 * w0 / wt, 100 * w1 / wt, 100 * w2 / wt,
            mma_cyc, sh.a_stages, sh.b_stages, sh.bres ? " (B resident)" : "");
  }
  return GG_OK;
}

// Fill the stage plan: B resident (only with a single N tile) if it fits beside
// >= 3 A stages, else a B ring; A stages = as many as fit (<= kSpanMaxStages).
static bool plan_span(SpanShape& sh, int bn, int rb, int taps, bool single_ntile, int reserve = 0) {
  // several boxes: multiples of 8 rows so each box starts on a swizzle atom
  sh.boxes = (sh.span_rows + 255) / 256;
  sh.box_rows = sh.boxes == 1 ? sh.span_rows : ((sh.span_rows + sh.boxes - 1) / sh.boxes + 7) / 8 * 8;
  sh.a_stage_bytes = (sh.boxes * sh.box_rows * rb + 1023) / 1024 * 1024;
  const int nkb = sh.C / (rb / 2) * taps;
  const int avail = kSpanSmemMax - 2048 - reserve;
  const int b_all = nkb * bn * rb;
  if (single_ntile && b_all + 3 * sh.a_stage_bytes <= avail) {   // one N tile: slab fixed
    sh.bres = 1;
    sh.b_stages = 1;
    sh.a_stages = (avail - b_all) / sh.a_stage_bytes;
  } else {
    // B ring: one tap slab (BN x 64 ch) is consumed every 4 * MT MMAs (~512
    // cycles) while an A span lasts all nine taps of a channel block, so the
    // smem goes to B depth (bytes in flight against L2 latency under load):
    // A double-buffered, B as deep as the rest allows.
    static const int a_env = getenv("GG_SPAN_ASTAGES") ? atoi(getenv("GG_SPAN_ASTAGES")) : 0;
    const int a_want = a_env > 1 ? a_env : 2;
    sh.bres = 0;
    sh.a_stages = a_want;
    const int bmax = (avail - a_want * sh.a_stage_bytes) / (bn * rb);
    sh.b_stages = bmax < kSpanMaxStages ? bmax : kSpanMaxStages;
    if (sh.b_stages < 2) {
      sh.b_stages = 2;
      sh.a_stages = (avail - 2 * bn * rb) / sh.a_stage_bytes;
    }
  }
  if (sh.a_stages > kSpanMaxStages) sh.a_stages = kSpanMaxStages;
  return sh.a_stages >= 2 && sh.b_stages >= 1;
}

// ---------------------------------------------------------------------------
// Stem conv + 3x3/2 max pool in one kernel (ResNet-18 conv1 / bn1 / relu / maxpool).
//
// The stem's 112 x 112 x 64 output (103 MB at batch 64) only feeds the max pool,
// so writing it and reading it back is pure HBM/L2 traffic.  Here a tile is TWO
// stem output rows (n, h) and (n, h + 1), h even: the 128 accumulator lanes are
// w = 0..127 (w >= Ws discarded) and the 128 accumulator columns are
// [row h: 64 channels | row h + 1: 64 channels].  Output row h + 1's tap (r, s)
// reads the same padded pixels as row h's tap (r + 1, s), so each of the 5 x 4
// row/column shifts (r', s) of the A span is ONE N = 128 MMA whose B slab is
// [W(r', s) ; W(r' - 1, s)] (zero halves at r' = 4 / r' = 0): 20 MMAs per two
// rows instead of 32 N = 64 ones — an M = 128, K = 16 MMA takes ~64 tensor cycles
// at N = 64 and N = 128 alike (tools/mma_bench.cu), so N = 64 wastes half the
// pipe.  The two B halves are TMA boxes of the [64, 256] weight matrix; the A
// span starts at the row's first padded pixel, rounded down to an 8-row swizzle
// atom (the descriptor carries the remainder).  Each CTA owns a contiguous band
// of pool rows g = n * Ho + ho; tile (2ho, 2ho + 1) completes pool row ho with
// the previous tile's row 2ho - 1 (a register partial), plus one extra tile
// (2ho0 - 2, 2ho0 - 1) at a band start inside an image:
//   epilogue phase 1: bias + ReLU + bf16 of both rows into swizzled smem rows
//                     (double buffered), one named barrier;
//   epilogue phase 2: horizontal 3-max at stride 2 from smem, vertical 3-max with
//                     the partial (thread -> (wo, 8-channel group) fixed), store.
// Max is order-independent and bf16 rounding monotonic, so the pooled values are
// identical to stem -> bf16 -> gg_maxpool3x3s2 (tests/test_resnet_gpu.py).
struct StemPoolShape {
  int N, Hs, Ws, Hp, Wp, Ho, Wo;
  int span_rows;      // 128 + 4 * Wp + 3 + 7: a row pair's span, atom-aligned start
  int a_stage_bytes;
  int a_stages;
  int out_pad;        // 0: dense [N, Ho, Wo, 64]; 2: shared-border layout
};

constexpr int kStemShifts = 20;                // (r', s): r' = 0..4, s = 0..3
constexpr int kStemBSlab = 128 * 32;           // one shift's B: 128 rows x 16 ch

struct StemTile { int n, h; bool pre; };

__device__ __forceinline__ uint32_t bmax2(uint32_t a, uint32_t b) {   // packed bf16x2 max (exact)
  act2_t r = __hmax2(*reinterpret_cast<act2_t*>(&a), *reinterpret_cast<act2_t*>(&b));
  return *reinterpret_cast<uint32_t*>(&r);
}

// Tile i of the CTA owning pool rows [g0, g1): image, first (even) stem row
__device__ __forceinline__ StemTile stem_tile(int i, int g0, int pre, int Ho) {
  StemTile t;
  t.pre = pre && i == 0;
  const int g = t.pre ? g0 : g0 + i - pre;
  t.n = g / Ho;
  t.h = 2 * (g - t.n * Ho) - (t.pre ? 2 : 0);
  return t;
}

__global__ void __launch_bounds__(kSpanThreads, 1)
    stem_pool_span(const __grid_constant__ CUtensorMap map_w, StemPoolShape sh,
                   const act_t* __restrict__ x16, const float* __restrict__ bias,
                   act_t* __restrict__ y, const int32_t* count) {
  constexpr int RB = 32, NACC = 4, ACC_COLS = 128;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_align1k(smem_raw);
  const int AST = sh.a_stages;
  uint8_t* a_base = smem;
  uint8_t* b_base = smem + AST * sh.a_stage_bytes;
  uint8_t* rowbuf = b_base + kStemShifts * kStemBSlab;   // epilogue column-exchange slots (1 KB)
  uint64_t* bars = reinterpret_cast<uint64_t*>(rowbuf + 1024);
  uint64_t* a_full = bars;
  uint64_t* a_empty = a_full + kSpanMaxStages;
  uint64_t* acc_full = a_empty + kSpanMaxStages;
  uint64_t* acc_empty = acc_full + NACC;
  uint64_t* b_full = acc_empty + NACC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(b_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  griddep_launch();
  if (threadIdx.x == 0) {
    for (int i = 0; i < AST; ++i) {
      mbar_init(&a_full[i], 1);
      mbar_init(&a_empty[i], 1);
    }
    for (int i = 0; i < NACC; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], kSpanEpiWarps);
    }
    mbar_init(b_full, 1);
    fence_mbar_init();
    tma_prefetch(&map_w);
  }
  if (warp == 1) tmem_alloc(tmem_slot, NACC * ACC_COLS);
  __syncthreads();
  // weights do not depend on the predecessor: load them before the wait.  Shift
  // (r', s): rows 0-63 = tap (r', s) for row h, rows 64-127 = tap (r' - 1, s) for h + 1
  if (warp == 0 && lane == 0) {
    mbar_expect_tx(b_full, 32 * 64 * RB);
    for (int j = 0; j < kStemShifts; ++j) {
      const int rr = j >> 2, s = j & 3;
      if (rr <= 3) tma_load_2d(b_base + j * kStemBSlab, &map_w, b_full, (rr * 4 + s) * 16, 0);
      if (rr >= 1) tma_load_2d(b_base + j * kStemBSlab + 64 * RB, &map_w, b_full, ((rr - 1) * 4 + s) * 16, 0);
    }
  } else if (warp >= 2) {   // the zero halves: top of r' = 4, bottom of r' = 0
    const int e = threadIdx.x - 64;   // 256 threads x 16 B x 4 = 16 KB
    for (int k = e; k < 1024; k += 256) {
      const int j = k >> 7, off = (k & 127) * 16;   // 8 half-slabs of 2 KB
      uint8_t* p = j < 4 ? b_base + (16 + j) * kStemBSlab + off : b_base + (j - 4) * kStemBSlab + 64 * RB + off;
      *reinterpret_cast<uint4*>(p) = make_uint4(0, 0, 0, 0);
    }
    fence_proxy_async_smem();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  griddep_wait();
  const int n_eff = count ? min(sh.N, __ldg(count)) : sh.N;
  const int total = n_eff * sh.Ho;   // pool rows
  const int g0 = (int)((int64_t)blockIdx.x * total / gridDim.x);
  const int g1 = (int)((int64_t)(blockIdx.x + 1) * total / gridDim.x);
  const int pre = (g1 > g0 && g0 % sh.Ho != 0) ? 1 : 0;
  const int ntiles = g1 > g0 ? pre + (g1 - g0) : 0;
  const int64_t rows_all = (int64_t)sh.N * sh.Hp * sh.Wp;

  if (warp == 0) {
    if (lane == 0) {
      for (int i = 0; i < ntiles; ++i) {
        const StemTile t = stem_tile(i, g0, pre, sh.Ho);
        const int as = i % AST;
        mbar_wait_sleep(&a_empty[as], ((i / AST) & 1) ^ 1);
        // output (h, w) reads padded input (h + r, w + s): the span of the pair starts at
        // padded pixel (n, h, 0); the 16-channel input is stored pre-swizzled (SW32), so
        // a linear copy from an 8-row-aligned start reproduces the swizzled image
        const int64_t m0 = ((int64_t)t.n * sh.Hp + t.h) * sh.Wp;
        const int64_t m0a = m0 & ~int64_t(7);
        const int64_t left = rows_all - m0a;
        const int rows = left < sh.span_rows ? (int)left : sh.span_rows;
        mbar_expect_tx(&a_full[as], rows * RB);
        bulk_load(a_base + as * sh.a_stage_bytes, x16 + m0a * 16, rows * RB, &a_full[as]);
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = idesc_act_f32(128, ACC_COLS);
    uint64_t sh_off[kStemShifts];
#pragma unroll
    for (int j = 0; j < kStemShifts; ++j) sh_off[j] = (uint64_t)(((j >> 2) * sh.Wp + (j & 3)) * (RB / 16));
    mbar_wait(b_full, 0);
    const uint64_t bdesc = sdesc_k_sw32(smem_u32(b_base));
    const uint64_t a_desc0 = sdesc_k_sw32(smem_u32(a_base));
    const uint64_t a_stage_d = (uint64_t)(sh.a_stage_bytes >> 4);
    int as = 0;
    uint32_t aph = 0;
    for (int i = 0; i < ntiles; ++i) {
      const StemTile t = stem_tile(i, g0, pre, sh.Ho);
      const int acc = i % NACC;
      mbar_wait(&acc_empty[acc], ((i / NACC) & 1) ^ 1);
      mbar_wait(&a_full[as], aph);
      tc_fence_after();
      const int64_t m0 = ((int64_t)t.n * sh.Hp + t.h) * sh.Wp;
      const uint64_t ad = a_desc0 + (uint64_t)as * a_stage_d + (uint64_t)((m0 & 7) * (RB / 16));
      const int as_now = as;
      if (++as == AST) {
        as = 0;
        aph ^= 1;
      }
      if (elect_one_sync()) {
#pragma unroll
        for (int j = 0; j < kStemShifts; ++j)
          umma_bf16(tmem_base + acc * ACC_COLS, ad + sh_off[j], bdesc + (uint64_t)(j * (kStemBSlab >> 4)), idesc,
                    j != 0);
        umma_commit(&a_empty[as_now]);
        umma_commit(&acc_full[acc]);
      }
      __syncwarp();
    }
  } else {
    // warp (quarter q, channel half c): lanes w = 32q + lane, channels 32c..32c+31 of
    // both rows.  Pool vertically in registers first (rows 2ho - 1 | 2ho | 2ho + 1:
    // the previous tile's second row is the register partial), then horizontally
    // across lanes by shuffles; lane 0 takes column w - 1 from the previous quarter's
    // lane 31 through a 64-byte smem slot.  No staging of the rows in shared memory
    // (whose bandwidth the N = 128 MMAs nearly saturate).
    const int quarter = warp & 3, c = (warp - 2) >> 2;
    const int w = quarter * 32 + lane;   // this lane's stem column
    uint32_t* xch = reinterpret_cast<uint32_t*>(rowbuf);   // [2 bufs][2 halves][4 quarters][16 words]
    float bz[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) bz[i] = __ldg(bias + c * 32 + i);
    uint32_t part[16];   // stem row 2ho - 1 at (w, this half's channels), bf16x2
    for (int i = 0; i < ntiles; ++i) {
      const StemTile t = stem_tile(i, g0, pre, sh.Ho);
      const int acc = i % NACC;
      mbar_wait_sleep(&acc_full[acc], (i / NACC) & 1);
      tc_fence_after();
      uint32_t r0[32], r1[32];
      const uint32_t ta = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * ACC_COLS + c * 32;
      tmem_ld_32x32b_x32(ta, r0);        // row h
      tmem_ld_32x32b_x32(ta + 64, r1);   // row h + 1
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[acc]);
      uint32_t vm[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const uint32_t a0 = pack_act(fmaxf(__uint_as_float(r0[2 * e]) + bz[2 * e], 0.0f),
                                      fmaxf(__uint_as_float(r0[2 * e + 1]) + bz[2 * e + 1], 0.0f));
        const uint32_t a1 = pack_act(fmaxf(__uint_as_float(r1[2 * e]) + bz[2 * e], 0.0f),
                                      fmaxf(__uint_as_float(r1[2 * e + 1]) + bz[2 * e + 1], 0.0f));
        uint32_t v = bmax2(a0, a1);
        if (t.h != 0) v = bmax2(v, part[e]);   // no stem row above row 0
        vm[e] = v;
        part[e] = a1;
      }
      if (t.pre) continue;   // band-start tile: only the partial (row 2ho0 - 1)
      uint32_t* slot = xch + (((i & 1) * 2 + c) * 4) * 16;
      if (lane == 31 && quarter < 3) {
#pragma unroll
        for (int e = 0; e < 16; e += 4)
          *reinterpret_cast<uint4*>(slot + quarter * 16 + e) = make_uint4(vm[e], vm[e + 1], vm[e + 2], vm[e + 3]);
      }
      // the exchange stays within a channel half: one named barrier per half (4 warps)
      asm volatile("bar.sync %0, 128;" ::"r"(1 + c) : "memory");
      uint32_t o[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const uint32_t right = __shfl_down_sync(0xffffffffu, vm[e], 1);
        uint32_t left = __shfl_up_sync(0xffffffffu, vm[e], 1);
        if (lane == 0) left = quarter > 0 ? slot[(quarter - 1) * 16 + e] : vm[e];   // w = 0: no column -1
        o[e] = bmax2(bmax2(left, vm[e]), right);
      }
      const int wo = w >> 1;
      if (!(lane & 1) && wo < sh.Wo) {
        const int ho = t.h >> 1;
        const int64_t oi = sh.out_pad == 2
                               ? (int64_t)(sh.Wo + 2) + ((int64_t)t.n * (sh.Ho + 1) + ho) * (sh.Wo + 1) + wo
                               : ((int64_t)t.n * sh.Ho + ho) * sh.Wo + wo;
        uint4* dst = reinterpret_cast<uint4*>(y + oi * 64 + c * 32);
#pragma unroll
        for (int e = 0; e < 16; e += 4) dst[e / 4] = make_uint4(o[e], o[e + 1], o[e + 2], o[e + 3]);
      }
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, NACC * ACC_COLS);
  }
}


// ---------------------------------------------------------------------------
// Pixel-pair span convolution: 3x3 / 1 with C = Cout = 64 (ResNet-18 layer 1).
//
// An M = 128, K = 16 MMA costs the tensor pipe ~64 cycles at N = 64 and N = 128
// alike (tools/mma_bench.cu), so the N = 64 span conv runs the pipe at half rate.
// Here an accumulator row (TMEM lane) is a PAIR of consecutive padded pixels:
// lane i of a tile owns window origins m = 2(q + i) + e, e in {0, 1}, and its 128
// columns are [e = 0: 64 channels | e = 1: 64 channels] — exactly the 256 contiguous
// output bytes of the pixel pair.  The activations are read as a [pixels / 2, 128]
// matrix (two 64-channel K halves per pair row).  Tap (r, s) of slot e reads pixel
// 2(q + i) + r*Wp + j with j = e + s in 0..3, i.e. pair row q + i + P and K half h
// with P = (r*Wp + j) >> 1, h = (r*Wp + j) & 1 — the same for both slots.  So per
// kernel row r there are four A operands (j = 0..3), each ONE row-shifted view of
// the span, and j's B operand holds W(r, j - e) for the slots where 0 <= j - e <= 2:
//   j = 0: [W(r,0) | -]      N = 64 into columns 0..63
//   j = 1: [W(r,1) | W(r,0)] N = 128
//   j = 2: [W(r,2) | W(r,1)] N = 128
//   j = 3: [- | W(r,2)]      N = 64 into columns 64..127
// With the row's three tap slabs stacked in shared memory as [W(r,2); W(r,1);
// W(r,0)] (64 N-rows each, K-major SW128), every B operand is a contiguous run of
// that stack (j = 2: rows 0..127, j = 1: rows 64..191, j = 0: rows 128..191, j = 3:
// rows 0..63) — the weight slab is the unmodified [64, 9 * 64] matrix, loaded as
// nine 64 x 64 TMA boxes.  48 MMAs per 256 outputs instead of 72 N = 64 ones.
// Needs Wp odd (the shared-border layout) so the output offset Wp + 1 is a whole
// number of pairs.  Epilogue as conv_span_tcgen05's TMA path, in pair rows.
__global__ void __launch_bounds__(kSpanThreads, 1)
    conv_span_px2(const __grid_constant__ CUtensorMap map_x, const __grid_constant__ CUtensorMap map_w,
                  const __grid_constant__ CUtensorMap map_out, const __grid_constant__ CUtensorMap map_res,
                  SpanShape sh, SpanEpi ep) {
  constexpr int ACC_COLS = 128, NACC = 4;
  constexpr int TAP_BYTES = 64 * 128;           // one 64 x 64 weight box
  constexpr int B_TOTAL = 9 * TAP_BYTES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_align1k(smem_raw);
  const int AST = sh.a_stages;
  const int half_bytes = sh.a_stage_bytes / 2;
  uint8_t* a_base = smem;
  uint8_t* b_base = smem + AST * sh.a_stage_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(b_base + B_TOTAL);
  uint64_t* a_full = bars;
  uint64_t* a_empty = a_full + kSpanMaxStages;
  uint64_t* acc_full = a_empty + kSpanMaxStages;
  uint64_t* acc_empty = acc_full + NACC;
  uint64_t* bres_full = acc_empty + NACC;
  uint64_t* res_full = bres_full + 1;      // [8 warps][2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(res_full + 2 * kSpanEpiWarps);
  uint8_t* stg_base = smem_align1k(reinterpret_cast<uint8_t*>(bars) + 1024);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  griddep_launch();
  const int img = sh.Hp * sh.Wp;
  if (threadIdx.x == 0) {
    for (int i = 0; i < AST; ++i) {
      mbar_init(&a_full[i], 1);
      mbar_init(&a_empty[i], 1);
    }
    for (int i = 0; i < NACC; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], kSpanEpiWarps);
    }
    mbar_init(bres_full, 1);
    for (int i = 0; i < 2 * kSpanEpiWarps; ++i) mbar_init(&res_full[i], 1);
    fence_mbar_init();
    tma_prefetch(&map_x);
    tma_prefetch(&map_w);
    tma_prefetch(&map_out);
    if (ep.residual) tma_prefetch(&map_res);
  }
  if (warp == 1) tmem_alloc(tmem_slot, NACC * ACC_COLS);
  const int tiles_max = (sh.N * img + 255) / 256;
  const bool b_loaded = tiles_max > (int)blockIdx.x;
  // the weights do not depend on the predecessor: row r's stack [W(r,2); W(r,1); W(r,0)]
  if (warp == 0 && lane == 0 && b_loaded) {
    mbar_expect_tx(bres_full, B_TOTAL);
    for (int r = 0; r < 3; ++r)
      for (int k = 0; k < 3; ++k)
        tma_load_2d(b_base + (r * 3 + k) * TAP_BYTES, &map_w, bres_full, (r * 3 + 2 - k) * 64, 0);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  griddep_wait();
  const int n_eff = ep.count ? min(sh.N, __ldg(ep.count)) : sh.N;
  const int Mtot = n_eff * img;
  const int num_tiles = (Mtot + 255) / 256;

  if (warp == 0) {
    if (lane == 0) {
      int as = 0;
      uint32_t aph = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        mbar_wait_sleep(&a_empty[as], aph ^ 1);
        uint8_t* sa = a_base + as * sh.a_stage_bytes;
        mbar_expect_tx(&a_full[as], 2 * sh.box_rows * 128);
        tma_load_2d(sa, &map_x, &a_full[as], 0, tile * 128);
        tma_load_2d(sa + half_bytes, &map_x, &a_full[as], 64, tile * 128);
        if (++as == AST) {
          as = 0;
          aph ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc128 = idesc_act_f32(128, 128);
    constexpr uint32_t idesc64 = idesc_act_f32(128, 64);
    // per (r, j): A offset (16-B units: K half + pair-row shift), B offset, N, column
    uint32_t a_off[12];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int v = r * sh.Wp + j;
        a_off[r * 4 + j] = (uint32_t)((v & 1) * (half_bytes >> 4) + (v >> 1) * 8);
      }
    if (b_loaded) mbar_wait(bres_full, 0);
    const uint64_t b_desc0 = sdesc_k_sw128(smem_u32(b_base));
    const uint64_t a_desc0 = sdesc_k_sw128(smem_u32(a_base));
    const uint64_t a_stage_d = (uint64_t)(sh.a_stage_bytes >> 4);
    int as = 0, t = 0;
    uint32_t aph = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++t) {
      const int acc = t % NACC;
      mbar_wait(&acc_empty[acc], ((t / NACC) & 1) ^ 1);
      tc_fence_after();
      const uint32_t d = tmem_base + acc * ACC_COLS;
      mbar_wait(&a_full[as], aph);
      tc_fence_after();
      const uint64_t ad = a_desc0 + (uint64_t)as * a_stage_d;
      const int as_now = as;
      if (++as == AST) {
        as = 0;
        aph ^= 1;
      }
      if (elect_one_sync()) {
#pragma unroll
        for (int r = 0; r < 3; ++r) {
          const uint64_t bs = b_desc0 + (uint64_t)(r * 3 * (TAP_BYTES >> 4));
          // j = 1 first: on r = 0 its N = 128 MMA initialises all 128 columns
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            umma_bf16(d, ad + a_off[r * 4 + 1] + kk * 2, bs + 64 * 8 + kk * 2, idesc128, (r | kk) != 0);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            umma_bf16(d, ad + a_off[r * 4 + 0] + kk * 2, bs + 128 * 8 + kk * 2, idesc64, 1);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            umma_bf16(d, ad + a_off[r * 4 + 2] + kk * 2, bs + kk * 2, idesc128, 1);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            umma_bf16(d + 64, ad + a_off[r * 4 + 3] + kk * 2, bs + kk * 2, idesc64, 1);
        }
        umma_commit(&a_empty[as_now]);
        umma_commit(&acc_full[acc]);
      }
      __syncwarp();
    }
  } else {
    // warp w: TMEM lane quarter w % 4, slot e = (w - 2) / 4 (columns e * 64 .. e * 64 + 63)
    const int quarter = warp & 3;
    const int e = (warp - 2) >> 2;
    uint8_t* stg = stg_base + (warp - 2) * 4096;
    uint64_t* rb = res_full + (warp - 2) * 2;
    uint32_t rph[2] = {0, 0};
    const bool has_res = ep.residual != nullptr;
    const int sw = (lane >> 1) & 3;
    const int out_shift = (sh.Wp + 1) >> 1;   // output position m + Wp + 1, in pairs
    int t = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++t) {
      const int acc = t % NACC;
      const uint32_t tbase = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * ACC_COLS + e * 64;
      const int pw = tile * 128 + quarter * 32;          // the warp's first pair row
      const int orow0 = pw + out_shift;
      const bool any = 2 * pw < Mtot;
      const int m = 2 * (pw + lane) + e;                  // this lane's window origin
      const int nimg = m / img;
      const int within = m - nimg * img;
      const int h = within / sh.Wp, w = within - h * sh.Wp;
      const bool real = m < Mtot && h < sh.Ho && w < sh.Wo;
      // staging buffer c for chunk c; with a residual both boxes are requested up
      // front (their latency overlaps the accumulator wait and chunk 0's math)
      if (has_res && any && lane == 0) {
        bulk_wait_read<0>();   // the previous tile's stores have read both buffers
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          mbar_expect_tx(&rb[c], 2048);
          tma_load_2d(stg + c * 2048, &map_res, &rb[c], e * 64 + 32 * c, orow0);
        }
      }
      __syncwarp();
      mbar_wait_sleep(&acc_full[acc], (t / NACC) & 1);
      tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < 2; ++c) {
        const int bsel = c;
        uint8_t* buf = stg + bsel * 2048;
        const int pcol = e * 64 + 32 * c;                 // column in the pair row
        if (!has_res && any && lane == 0) bulk_wait_read<1>();   // the store two chunks back
        __syncwarp();
        uint32_t r[32];
        tmem_ld_32x32b_x32(tbase + 32 * c, r);
        tmem_ld_wait();
        if (!any) continue;
        uint4* myrow = reinterpret_cast<uint4*>(buf + lane * 64);
        float v[32];
        if (has_res) {
          mbar_wait(&rb[bsel], rph[bsel]);
          rph[bsel] ^= 1;
        }
        if (real) {
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            const float4 bb = __ldg(reinterpret_cast<const float4*>(ep.bias + 32 * c + i));
            v[i] = __uint_as_float(r[i]) + bb.x;
            v[i + 1] = __uint_as_float(r[i + 1]) + bb.y;
            v[i + 2] = __uint_as_float(r[i + 2]) + bb.z;
            v[i + 3] = __uint_as_float(r[i + 3]) + bb.w;
          }
          if (has_res) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const uint4 u = myrow[q ^ sw];
              const act2_t* h2 = reinterpret_cast<const act2_t*>(&u);
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const float2 f = act2_to_float2(h2[k]);
                v[q * 8 + 2 * k] += f.x;
                v[q * 8 + 2 * k + 1] += f.y;
              }
            }
          }
          if (ep.relu) {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = fmaxf(v[i], 0.0f);
          }
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = 0.0f;      // padding positions stay zero
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 u;
          u.x = pack_act(v[q * 8 + 0], v[q * 8 + 1]);
          u.y = pack_act(v[q * 8 + 2], v[q * 8 + 3]);
          u.z = pack_act(v[q * 8 + 4], v[q * 8 + 5]);
          u.w = pack_act(v[q * 8 + 6], v[q * 8 + 7]);
          myrow[q ^ sw] = u;
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_2d(&map_out, buf, pcol, orow0);
          bulk_commit();
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[acc]);
    }
    if (lane == 0) bulk_wait<0>();
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, NACC * ACC_COLS);
  }
}

// Launch conv_span_px2 for a shared-border 3x3 / 1 conv with C = Cout = 64 (Wp odd).
// Returns GG_ERR_UNSUPPORTED when the shape does not qualify (the caller falls back).
static int launch_span_px2(const void* x, const void* w, const float* bias, const void* residual,
                           int relu, void* y, const int32_t* count_dev, SpanShape sh, cudaStream_t s) {
  if (sh.C != 64 || sh.Cout != 64 || !(sh.Wp & 1)) return GG_ERR_UNSUPPORTED;
  const int64_t Mtot = (int64_t)sh.N * sh.Hp * sh.Wp;
  sh.span_rows = 128 + sh.Wp + 1;                    // pair rows: max shift (2 Wp + 3) >> 1
  if (sh.span_rows > 256) return GG_ERR_UNSUPPORTED;
  sh.boxes = 1;
  sh.box_rows = sh.span_rows;
  sh.a_stage_bytes = 2 * ((sh.span_rows * 128 + 1023) / 1024 * 1024);
  sh.bres = 1;
  sh.b_stages = 1;
  const int fixed = 9 * 64 * 128 + 2048 + kSpanStgBytes;
  sh.a_stages = (kSpanSmemMax - fixed) / sh.a_stage_bytes;
  if (sh.a_stages > kSpanMaxStages) sh.a_stages = kSpanMaxStages;
  if (sh.a_stages < 2) return GG_ERR_UNSUPPORTED;
  // pair rows cover pixel Mtot when Mtot is odd: the buffers hold the W + 2-pixel
  // margin beyond the N images (shared-border layout), and that pixel is a border
  // column position (written as zero)
  const int64_t prows = (Mtot + 1) / 2;
  CUtensorMap mx, mw, mo, mr;
  int rc = make_map_span(&mx, x, prows, 128, 64, sh.box_rows);
  if (!rc) rc = make_map_span(&mw, w, 64, 9 * 64, 64, 64);
  if (!rc) rc = make_map_box32(&mo, y, prows, 128);
  if (!rc && residual) rc = make_map_box32(&mr, residual, prows, 128);
  if (rc) return rc;
  auto kern = conv_span_px2;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSpanSmemMax) != cudaSuccess)
      return GG_ERR_CUDA;
    attr = true;
  }
  SpanEpi ep{reinterpret_cast<act_t*>(y), bias, reinterpret_cast<const act_t*>(residual), relu, count_dev,
             nullptr, nullptr, 0, 1, StreamK{nullptr, nullptr, 0}};
  const int smem = sh.a_stages * sh.a_stage_bytes + fixed;
  const int tiles = (int)((Mtot + 255) / 256);
  const int grid = tiles < num_sms() ? tiles : num_sms();
  if (launch_pdl(kern, dim3(grid), dim3(kSpanThreads), smem, s, mx, mw, mo, residual ? mr : mo, sh, ep) !=
      cudaSuccess)
    return GG_ERR_CUDA;
  return GG_OK;
}

}  // namespace gg

using namespace gg;

// border 2: zero-bordered [N, H+2, W+2, C]; border 1: shared-border layout (one zero
// row / column per image, [N, H+1, W+1, C] after a W+2-row zero margin) — the left
// and top neighbours of an image's first column / row are the previous column's /
// image's zero row, so 3x3 taps stay uniform row shifts with Wp = W + 1.
static int conv3x3_span(const void* x, int32_t N, int32_t H, int32_t W, int32_t C, const void* w,
                        int32_t Cout, const float* bias, const void* residual, int32_t relu, void* y,
                        const int32_t* count_dev, void* stream, int border) {
  if (!x || !w || !y || !bias || N <= 0 || H <= 0 || W <= 0) return GG_ERR_INVALID_ARGUMENT;
  if (C % 64 || Cout % 64) return GG_ERR_UNSUPPORTED;
  SpanShape sh;
  sh.N = N; sh.H = H; sh.W = W; sh.C = C; sh.Cout = Cout;
  sh.Hp = H + border; sh.Wp = W + border;
  sh.Ho = H; sh.Wo = W;
  const int64_t Mtot = (int64_t)N * sh.Hp * sh.Wp;
  // Tile shape (BN x 128*MT) by a per-SM time model: MMA cycles per tile
  // (tools/mma_bench.cu: 48 / 64 / 128 cycles per K=16 step at N = 64/128/256)
  // vs the SM's operand ingress (~40 B/cycle: B slabs unless resident + A
  // spans), tiles per CTA, plus the last tile's epilogue and the resident-B
  // prologue, which nothing overlaps.
  // CTA pairs (cta_group::2, M = 256 over two SMs) for Cout >= 128: half the
  // smem operand reads per MMA and half the weight stream per SM (see
  // conv_span_pair).  GG_SPAN_PAIR=0 keeps single-CTA tiles.
  static const bool no_pair = getenv("GG_SPAN_PAIR") && atoi(getenv("GG_SPAN_PAIR")) == 0;
  // N = 64 pairs (layer 1) measured slower than single-CTA tiles (GG_SPAN_PAIR64=1 opts in)
  static const bool pair64 = getenv("GG_SPAN_PAIR64") && atoi(getenv("GG_SPAN_PAIR64")) == 1;
  // C = Cout = 64 on the shared-border layout: pixel-pair tiles (N = 128 MMAs, see
  // conv_span_px2); GG_SPAN_PX2=0 keeps the N = 64 span conv
  static const bool no_px2 = getenv("GG_SPAN_PX2") && atoi(getenv("GG_SPAN_PX2")) == 0;
  if (!no_px2 && border == 1 && C == 64 && Cout == 64 && !pair64 && !getenv("GG_SPAN_TILE")) {
    const int rc = launch_span_px2(x, w, bias, residual, relu, y, count_dev, sh, gg_stream(stream));
    if (rc != GG_ERR_UNSUPPORTED) return rc;
  }
  if (!no_pair && (Cout % 128 == 0 || (Cout == 64 && pair64)) && !getenv("GG_SPAN_TILE")) {
    int bn = Cout % 256 == 0 ? 256 : Cout % 128 == 0 ? 128 : 64;
    if (bn == 256) {   // N = 128 pair tiles unless N = 256 finishes in strictly fewer rounds x width
      const int64_t mt = (Mtot + 255) / 256, P = num_sms() / 2;
      const int64_t r256 = (mt * (Cout / 256) + P - 1) / P, r128 = (mt * (Cout / 128) + P - 1) / P;
      // ties go to N = 128 (layer 3: 114 tiles in 2 rounds beat 57 in 1 once the issue
      // loop was lean — 17.5 vs 19.5 us — the second tile's MMAs overlap the first's
      // epilogue); GG_SPAN_PAIR_BN=128/256 forces a width
      static const int pair_bn = getenv("GG_SPAN_PAIR_BN") ? atoi(getenv("GG_SPAN_PAIR_BN")) : 0;
      if (pair_bn == 128 || (pair_bn != 256 && r128 * 128 <= r256 * 256)) bn = 128;
    }
    sh.span_rows = 128 + 2 * sh.Wp + 2;
    // coalesced TMA-box epilogue (GG_NO_TMA_EPI=1 keeps row-per-thread stores)
    static const bool no_tma_epi = getenv("GG_NO_TMA_EPI") != nullptr;
    const bool tma_epi = !no_tma_epi;
    if (sh.span_rows <= 1024 && plan_span(sh, bn / 2, 128, 9, bn == Cout, tma_epi ? kSpanStgBytes : 0)) {
      CUtensorMap mx, mw, mo, mr;
      int rc = make_map_span(&mx, x, Mtot, C, 64, sh.box_rows);
      if (!rc) rc = make_map_span(&mw, w, Cout, (int64_t)C * 9, 64, bn / 2);
      if (!rc && tma_epi) rc = make_map_box32(&mo, y, Mtot, Cout);
      if (!rc && tma_epi && residual) rc = make_map_box32(&mr, residual, Mtot, Cout);
      if (rc) return rc;
      SpanEpi ep{reinterpret_cast<act_t*>(y), bias,
                 reinterpret_cast<const act_t*>(residual), relu, count_dev, nullptr, nullptr, 0,
                 tma_epi ? 1 : 0, StreamK{nullptr, nullptr, 0}};
      cudaStream_t s = gg_stream(stream);
      // stream-K over (pair tile, channel block) for pair tiles that leave the last
      // wave mostly empty (layer 4: 42 tiles on 74 pairs).  Opt-in (GG_SPAN_SK=1):
      // correct and deterministic (test_span_pair_stream_k) but measured slower at
      // every ResNet-18 stage (e.g. layer 4: 39 vs 30 us per conv) — the partial
      // regions' global round trip and the per-item pipeline drains cost more than
      // the idle SMs of the data-parallel schedule.
      {
        const int64_t tiles = (Mtot + 255) / 256 * (Cout / bn);
        const int P = num_sms() / 2;
        const char* env = getenv("GG_SPAN_SK");
        const bool want = env && atoi(env) == 1;
        if (tma_epi && want && tiles * (C / 64) >= 2 * P) {
          bool ok = false;
          StreamK sk = streamk_workspace(s, (int64_t)P * 2 * 16 * 32 * (bn / 2), tiles * 16 * 2, ok);
          if (ok) ep.sk = sk;
        }
      }
      const CUtensorMap* po = tma_epi ? &mo : nullptr;
      const CUtensorMap* pr = tma_epi && residual ? &mr : nullptr;
      return bn == 256 ? launch_span_pair<256>(mx, mw, sh, ep, s, po, pr)
             : bn == 128 ? launch_span_pair<128>(mx, mw, sh, ep, s, po, pr)
                         : launch_span_pair<64>(mx, mw, sh, ep, s, po, pr);
    }
  }
  const int cblocks = C / 64;
  struct Cand { int bn, mt; };
  const Cand cands[] = {{64, 1}, {128, 1}, {256, 1}, {64, 2}, {128, 2}};
  int best_bn = 64, best_mt = 1;
  double best = 1e30;
  for (const Cand& cd : cands) {
    if (cd.bn > Cout || Cout % cd.bn) continue;
    SpanShape t = sh;
    t.span_rows = 128 * cd.mt + 2 * sh.Wp + 2;
    if (t.span_rows > 1024 || !plan_span(t, cd.bn, 128, 9, cd.bn == Cout)) continue;
    const int64_t tiles = (Mtot + 128 * cd.mt - 1) / (128 * cd.mt) * (Cout / cd.bn);
    const int64_t per_cta = (tiles + num_sms() - 1) / num_sms();
    const double cyc_k = cd.bn == 64 ? 48.0 : cd.bn / 2.0;
    const double mma = (double)cblocks * 9 * 4 * cd.mt * cyc_k;
    const double ingress = ((double)cblocks * t.boxes * t.box_rows * 128 +
                            (t.bres ? 0.0 : (double)cblocks * 9 * cd.bn * 128)) / 40.0;
    const double tile = mma > ingress ? mma : ingress;
    const double epi = cd.mt * (cd.bn / 64.0) * 700.0;
    const double pro = t.bres ? (double)cblocks * 9 * cd.bn * 128 / 40.0 : 0.0;
    const double tt = per_cta * tile + epi + pro;
    if (tt < best * 0.97) {
      best = tt;
      best_bn = cd.bn;
      best_mt = cd.mt;
    }
  }
  if (getenv("GG_SPAN_TILE")) {   // debug override "BN,MT"
    int a = 0, b = 0;
    if (sscanf(getenv("GG_SPAN_TILE"), "%d,%d", &a, &b) == 2 && a > 0 && Cout % a == 0 && (b == 1 || b == 2)) {
      best_bn = a;
      best_mt = b;
    }
  }
  sh.span_rows = 128 * best_mt + 2 * sh.Wp + 2;
  static const bool no_tma_epi1 = getenv("GG_NO_TMA_EPI") != nullptr;
  const bool tma1 = !no_tma_epi1;
  if (sh.span_rows > 1024 || !plan_span(sh, best_bn, 128, 9, best_bn == Cout, tma1 ? kSpanStgBytes : 0))
    return GG_ERR_UNSUPPORTED;
  CUtensorMap mx, mw, mo, mr;
  int rc = make_map_span(&mx, x, Mtot, C, 64, sh.box_rows);
  if (!rc) rc = make_map_span(&mw, w, Cout, (int64_t)C * 9, 64, best_bn);
  if (!rc && tma1) rc = make_map_box32(&mo, y, Mtot, Cout);
  if (!rc && tma1 && residual) rc = make_map_box32(&mr, residual, Mtot, Cout);
  if (rc) return rc;
  SpanEpi ep{reinterpret_cast<act_t*>(y), bias,
             reinterpret_cast<const act_t*>(residual), relu, count_dev, nullptr, nullptr, 0,
             tma1 ? 1 : 0, StreamK{nullptr, nullptr, 0}};
  cudaStream_t s = gg_stream(stream);
  const CUtensorMap* po = tma1 ? &mo : nullptr;
  const CUtensorMap* pr = tma1 && residual ? &mr : nullptr;
  switch (best_bn * 4 + best_mt) {
    case 256 * 4 + 1: return launch_span<256, 64, 3, false, 1>(mx, mw, sh, ep, s, po, pr);
    case 128 * 4 + 1: return launch_span<128, 64, 3, false, 1>(mx, mw, sh, ep, s, po, pr);
    case 128 * 4 + 2: return launch_span<128, 64, 3, false, 2>(mx, mw, sh, ep, s, po, pr);
    case 64 * 4 + 2: return launch_span<64, 64, 3, false, 2>(mx, mw, sh, ep, s, po, pr);
    default: return launch_span<64, 64, 3, false, 1>(mx, mw, sh, ep, s, po, pr);
  }
}

extern "C" int gg_conv3x3_padded(const void* x, int32_t N, int32_t H, int32_t W, int32_t C,
                                 const void* w, int32_t Cout, const float* bias,
                                 const void* residual, int32_t relu, void* y,
                                 const int32_t* count_dev, void* stream) {
  return conv3x3_span(x, N, H, W, C, w, Cout, bias, residual, relu, y, count_dev, stream, 2);
}

extern "C" int gg_conv3x3_shared(const void* x, int32_t N, int32_t H, int32_t W, int32_t C,
                                 const void* w, int32_t Cout, const float* bias,
                                 const void* residual, int32_t relu, void* y,
                                 const int32_t* count_dev, void* stream) {
  return conv3x3_span(x, N, H, W, C, w, Cout, bias, residual, relu, y, count_dev, stream, 1);
}

extern "C" int gg_stem_s2d_span(const void* x, int32_t N, int32_t Hs, int32_t Ws, const void* w,
                                int32_t Cout, const float* bias, int32_t relu, void* y,
                                const int32_t* count_dev, void* stream) {
  if (!x || !w || !y || !bias || N <= 0 || Hs <= 0 || Ws <= 0) return GG_ERR_INVALID_ARGUMENT;
  if (Cout != 64) return GG_ERR_UNSUPPORTED;
  SpanShape sh;
  sh.N = N; sh.H = Hs; sh.W = Ws; sh.C = 16; sh.Cout = Cout;
  sh.Hp = Hs + 3; sh.Wp = Ws + 3;   // space-to-depth input padded 2 before, 1 after
  sh.Ho = Hs; sh.Wo = Ws;
  sh.span_rows = 128 + 3 * sh.Wp + 3;
  if (sh.span_rows > 1024) return GG_ERR_UNSUPPORTED;
  if (!plan_span(sh, 64, 32, 16, true, kSpanStgBytes)) return GG_ERR_UNSUPPORTED;
  const int64_t Mtot = (int64_t)N * sh.Hp * sh.Wp;
  CUtensorMap mx, mw;
  int rc = make_map_span(&mx, x, Mtot, 16, 16, sh.box_rows);
  if (!rc) rc = make_map_span(&mw, w, Cout, 256, 16, 64);
  if (rc) return rc;
  SpanEpi ep{reinterpret_cast<act_t*>(y), bias, nullptr, relu, count_dev, nullptr,
             reinterpret_cast<const act_t*>(x), 0, 0, StreamK{nullptr, nullptr, 0}};
  if (reinterpret_cast<uintptr_t>(x) & 15) return GG_ERR_INVALID_ARGUMENT;
  // CTA-pair stem: correct but measured 94 us vs 59 us for single-CTA tiles
  // (N = 64 pair MMAs); GG_SPAN_PAIR64=1 opts in
  static const bool pair64 = getenv("GG_SPAN_PAIR64") && atoi(getenv("GG_SPAN_PAIR64")) == 1;
  if (pair64) {
    // CTA pair (M = 256 per MMA): the input is stored pre-swizzled (SW32), so the
    // span comes in through an unswizzled TMA map (a plain row copy, like the
    // single-CTA bulk copy) that can complete on the leader's barrier
    SpanShape sp = sh;
    if (!plan_span(sp, 32, 32, 16, true)) return GG_ERR_UNSUPPORTED;
    CUtensorMap mxp, mwp;
    rc = make_map_span(&mxp, x, Mtot, 16, 16, sp.box_rows, true);
    if (!rc) rc = make_map_span(&mwp, w, Cout, 256, 16, 32);
    if (rc) return rc;
    return launch_span_pair<64, 16, 4, true>(mxp, mwp, sp, ep, gg_stream(stream));
  }
  return launch_span<64, 16, 4, true, 1>(mx, mw, sh, ep, gg_stream(stream));
}

extern "C" int gg_stem_pool_span(const void* x, int32_t N, int32_t Hs, int32_t Ws, const void* w,
                                 int32_t Cout, const float* bias, void* y, int32_t out_pad,
                                 const int32_t* count_dev, void* stream) {
  if (!x || !w || !y || !bias || N <= 0 || Hs <= 0 || Ws <= 0) return GG_ERR_INVALID_ARGUMENT;
  if (reinterpret_cast<uintptr_t>(x) & 15) return GG_ERR_INVALID_ARGUMENT;
  if (Cout != 64 || (Hs & 1) || (Ws & 1) || Ws > 128 || (out_pad != 0 && out_pad != 2))
    return GG_ERR_UNSUPPORTED;
  StemPoolShape sh;
  sh.N = N; sh.Hs = Hs; sh.Ws = Ws;
  sh.Hp = Hs + 3; sh.Wp = Ws + 3;   // space-to-depth input padded 2 before, 1 after
  sh.Ho = Hs / 2; sh.Wo = Ws / 2;   // 3x3 / 2 / pad 1 over an even extent
  sh.out_pad = out_pad;
  sh.span_rows = 128 + 4 * sh.Wp + 3 + 7;
  sh.a_stage_bytes = (sh.span_rows * 32 + 1023) / 1024 * 1024;
  const int fixed = 1024 + kStemShifts * kStemBSlab + 1024 + 1024;
  sh.a_stages = (kSpanSmemMax - fixed) / sh.a_stage_bytes;
  if (sh.a_stages > 8) sh.a_stages = 8;
  if (sh.a_stages < 2) return GG_ERR_UNSUPPORTED;
  CUtensorMap mw;
  if (int rc = make_map_span(&mw, w, Cout, 256, 16, 64)) return rc;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(stem_pool_span, cudaFuncAttributeMaxDynamicSharedMemorySize, kSpanSmemMax) !=
        cudaSuccess)
      return GG_ERR_CUDA;
    attr = true;
  }
  const int smem = fixed + sh.a_stages * sh.a_stage_bytes;
  const int64_t rows = (int64_t)N * sh.Ho;
  const int grid = rows < num_sms() ? (int)rows : num_sms();
  if (launch_pdl(stem_pool_span, dim3(grid), dim3(kSpanThreads), smem, gg_stream(stream), mw, sh,
                 reinterpret_cast<const act_t*>(x), bias, reinterpret_cast<act_t*>(y),
                 count_dev) != cudaSuccess)
    return GG_ERR_CUDA;
  return GG_OK;
}
