// gg_attention.cu — DistilBERT self-attention (S = 128, head dim 64) on tcgen05.
//
// One CTA per (batch, head), 4 warps:
//   TMA  : Q [128 x 64], K [128 x 64] and V^T [64 x 128] (written transposed by
//          the QKV GEMM epilogue) into 128B-swizzled smem;
//   MMA 1: S = Q K^T (M=128, N=128, K=64) into TMEM columns [0, 128);
//   softmax: each thread owns one query row, reads its 128 scores with
//          tcgen05.ld, applies the key mask, exp(s - max) in fp32, writes the
//          unnormalized P row (bf16, <= 1) into the swizzled A-operand layout;
//   MMA 2: O = P V (M=128, N=64, K=128) into TMEM columns [128, 192);
//   epilogue: O / rowsum -> bf16 ctx[b*S + s, h*64 + d].
#include <cudaTypedefs.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>

#include "gg_common.cuh"
#include "gg_kernels.h"
#include "gg_tc.cuh"

namespace gg {
using namespace tc;

constexpr int kAttnS = 128;
constexpr int kAttnD = 64;
constexpr int kAttnThreads = 128;
// smem: Q [0,16K) K [16K,32K) V^T [32K,48K); P (2 x 16 KB key blocks) reuses
// Q+K once S = QK^T is in TMEM.  TMEM: 128 columns, S in [0,128), then O in
// [0,64) once every thread has read its S row.  48 KB + 128 columns -> 4 CTAs/SM.
constexpr int kOffQ = 0, kOffK = 16384, kOffV = 32768, kOffP = 0;
constexpr int kAttnSmem = 49152 + 64 + 1024;

__global__ void __launch_bounds__(kAttnThreads, 4)
    attention_tcgen05(const __grid_constant__ CUtensorMap map_q,
                      const __grid_constant__ CUtensorMap map_k,
                      const __grid_constant__ CUtensorMap map_vt, const int32_t* mask,
                      __nv_bfloat16* ctx, int64_t ldc, int heads, const int32_t* count) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_align1k(smem_raw);
  uint64_t* bar_load = reinterpret_cast<uint64_t*>(smem + 49152);
  uint64_t* bar_s = bar_load + 1;
  uint64_t* bar_o = bar_load + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar_load + 3);
  __shared__ float key_bias[kAttnS];   // 0 or -inf per key (attention mask)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int bh = blockIdx.x;
  const int b = bh / heads, h = bh % heads;

  griddep_launch();   // programmatic dependent launch: the successor's prologue may start
  if (threadIdx.x == 0) {
    mbar_init(bar_load, 1);
    mbar_init(bar_s, 1);
    mbar_init(bar_o, 1);
    fence_mbar_init();
    tma_prefetch(&map_q);
    tma_prefetch(&map_k);
    tma_prefetch(&map_vt);
  }
  griddep_wait();     // Q/K/V, the mask and the count follow the predecessor
  if (count && (int)(blockIdx.x / heads) >= __ldg(count)) return;  // dynamic batch (CTA-uniform)
  key_bias[threadIdx.x] = (mask && __ldg(mask + (int64_t)b * kAttnS + threadIdx.x) == 0) ? -INFINITY : 0.0f;
  if (warp == 0) tmem_alloc(tmem_slot, 128);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (threadIdx.x == 0) {
    mbar_expect_tx(bar_load, 16384 + 16384 + 2 * 8192);  // Q + K + V^T (two 64-key blocks)
    tma_load_2d(smem + kOffQ, &map_q, bar_load, 0, bh * kAttnS);
    tma_load_2d(smem + kOffK, &map_k, bar_load, 0, bh * kAttnS);
    tma_load_2d(smem + kOffV, &map_vt, bar_load, 0, bh * kAttnD);
    tma_load_2d(smem + kOffV + 8192, &map_vt, bar_load, 64, bh * kAttnD);
    mbar_wait(bar_load, 0);
    tc_fence_after();
    const uint32_t sq = smem_u32(smem + kOffQ), sk = smem_u32(smem + kOffK);
    constexpr uint32_t idesc_s = idesc_bf16_f32(128, 128);
#pragma unroll
    for (int kk = 0; kk < 4; ++kk)
      umma_bf16(tmem, sdesc_k_sw128(sq + kk * 32), sdesc_k_sw128(sk + kk * 32), idesc_s, kk != 0);
    umma_commit(bar_s);
  }

  // ---- softmax: thread = query row; two passes over S straight from TMEM ----
  const int row = warp * 32 + lane;
  const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
  mbar_wait(bar_s, 0);
  tc_fence_after();
  float mx = -INFINITY;
#pragma unroll
  for (int c = 0; c < kAttnS; c += 64) {   // two TMEM loads per wait
    uint32_t r[2][32];
    tmem_ld_32x32b_x32(trow + c, r[0]);
    tmem_ld_32x32b_x32(trow + c + 32, r[1]);
    tmem_ld_wait();
#pragma unroll
    for (int hh = 0; hh < 2; ++hh)
#pragma unroll
      for (int i = 0; i < 32; ++i) mx = fmaxf(mx, __uint_as_float(r[hh][i]) + key_bias[c + 32 * hh + i]);
  }
  const float mref = (mx == -INFINITY) ? 0.0f : mx;
  const float l2e = 1.4426950408889634f;
  float sum = 0.0f;
  // P row -> A operand (K-major, SW128): key block kb = j / 64, 16-byte chunk (j % 64) / 8
  uint8_t* prow = smem + kOffP + (row >> 3) * 1024 + (row & 7) * 128;
#pragma unroll
  for (int c = 0; c < kAttnS; c += 32) {
    uint32_t r[32];
    tmem_ld_32x32b_x32(trow + c, r);
    tmem_ld_wait();
    float e[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      e[i] = exp2f((__uint_as_float(r[i]) + key_bias[c + i] - mref) * l2e);
      sum += e[i];
    }
    const int kb = c / 64;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int chunk = (c % 64) / 8 + q;
      uint4 u;
      u.x = pack_bf16(e[8 * q + 0], e[8 * q + 1]);
      u.y = pack_bf16(e[8 * q + 2], e[8 * q + 3]);
      u.z = pack_bf16(e[8 * q + 4], e[8 * q + 5]);
      u.w = pack_bf16(e[8 * q + 6], e[8 * q + 7]);
      *reinterpret_cast<uint4*>(prow + kb * 16384 + ((chunk ^ (row & 7)) << 4)) = u;
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();   // every S row read, every P row written
  if (threadIdx.x == 0) {
    tc_fence_after();
    const uint32_t sp = smem_u32(smem + kOffP), sv = smem_u32(smem + kOffV);
    constexpr uint32_t idesc_o = idesc_bf16_f32(128, 64);
#pragma unroll
    for (int kb = 0; kb < 2; ++kb)
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        umma_bf16(tmem, sdesc_k_sw128(sp + kb * 16384 + kk * 32),
                  sdesc_k_sw128(sv + kb * 8192 + kk * 32), idesc_o, (kb | kk) != 0);
    umma_commit(bar_o);
  }
  mbar_wait(bar_o, 0);
  tc_fence_after();
  const float inv = 1.0f / sum;
  __nv_bfloat16* out = ctx + ((int64_t)b * kAttnS + row) * ldc + h * kAttnD;
#pragma unroll
  for (int c = 0; c < kAttnD; c += 32) {
    uint32_t r[32];
    tmem_ld_32x32b_x32(trow + c, r);
    tmem_ld_wait();
    uint4* dp = reinterpret_cast<uint4*>(out + c);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint4 u;
      u.x = pack_bf16(__uint_as_float(r[8 * q + 0]) * inv, __uint_as_float(r[8 * q + 1]) * inv);
      u.y = pack_bf16(__uint_as_float(r[8 * q + 2]) * inv, __uint_as_float(r[8 * q + 3]) * inv);
      u.z = pack_bf16(__uint_as_float(r[8 * q + 4]) * inv, __uint_as_float(r[8 * q + 5]) * inv);
      u.w = pack_bf16(__uint_as_float(r[8 * q + 6]) * inv, __uint_as_float(r[8 * q + 7]) * inv);
      dp[q] = u;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 128);
  }
}


// ---------------------------------------------------------------------------
// Persistent, warp-specialized attention: one CTA per SM walks the (batch,
// head) items c, c + grid, ... with every phase of consecutive items
// overlapped (the per-item kernel above serializes load -> QK^T -> softmax ->
// PV -> store inside one CTA and ran latency-bound at ~19 % occupancy):
//   warp 0     TMA producer: Q, K, V^T (+ the item's key-mask row) into one of
//              two 48 KB stages
//   warp 1     MMA issuer: S(t+1) = Q K^T is issued before O(t) = P(t) V, so the
//              tensor core works on the next item while the softmax runs
//   warps 2-5, 6-9  two compute groups, items alternating between them;
//              thread = query row.  softmax: the 128 scores of its row from
//              TMEM into registers, max, ex2, sum, unnormalized P row (bf16,
//              <= 1) into the group's swizzled A-operand buffer; epilogue
//              after O = P V: O row / sum -> bf16 -> SW128 staging tile -> one
//              TMA store of the [128 x 64] ctx box per item.  While one group
//              waits for its O, the other group's softmax runs.
// TMEM: S buffers [0, 256) and O buffers [256, 384), one of each per group.
constexpr int kApThreads = 320;
constexpr int kApStages = 3;                        // loads in flight per SM (HBM latency)
constexpr int kApStageBytes = 50176;                 // Q 16K | K 16K | V^T 16K | mask 512 (1 KB pad)
constexpr int kApOffStage = 0;
constexpr int kApOffP = kApStages * kApStageBytes;   // 2 x 32 KB (P, then the ctx staging tile)
constexpr int kApOffBar = kApOffP + 2 * 32768;
constexpr int kApSmem = kApOffBar + 256 + 1024;

__device__ __forceinline__ void named_bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__global__ void __launch_bounds__(kApThreads, 1)
    attention_persist(const __grid_constant__ CUtensorMap map_q,
                      const __grid_constant__ CUtensorMap map_k,
                      const __grid_constant__ CUtensorMap map_vt,
                      const __grid_constant__ CUtensorMap map_o, const int32_t* mask, int batch,
                      int heads, const int32_t* count, int dbg, gg_dep dep) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_align1k(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kApOffBar);
  uint64_t* full = bars;         // [3] stage loaded (tx bytes)
  uint64_t* empty = bars + 3;    // [3] stage free (MMA commit after O)
  uint64_t* s_full = bars + 6;   // [2] S in TMEM (MMA commit), per group
  uint64_t* s_empty = bars + 8;  // [2] S read by the group's 128 threads
  uint64_t* p_full = bars + 10;  // [2] P written by the group's 128 threads
  uint64_t* o_full = bars + 12;  // [2] O in TMEM (MMA commit)
  uint64_t* o_empty = bars + 14; // [2] O read by the group's 128 threads
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 16);
  int* cnt_slot = reinterpret_cast<int*>(bars + 17);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  griddep_launch();
  if (threadIdx.x == 0) {
    for (int i = 0; i < kApStages; ++i) {
      mbar_init(full + i, 1);
      mbar_init(empty + i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(s_full + i, 1);
      mbar_init(s_empty + i, 128);
      mbar_init(p_full + i, 128);
      mbar_init(o_full + i, 1);
      mbar_init(o_empty + i, 128);
    }
    fence_mbar_init();
    tma_prefetch(&map_q);
    tma_prefetch(&map_k);
    tma_prefetch(&map_vt);
    tma_prefetch(&map_o);
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (dep.wait) {
    // tile-level dependencies (gg_dep): the count once the chain has started;
    // each item waits for its sequence's QKV tiles below
    if (threadIdx.x == 0) {
      dep_wait_geq(dep.go, 1);
      *cnt_slot = count ? ld_relaxed_gpu(count) : batch;
    }
  } else {
    griddep_wait();     // Q/K/V, the mask and the count follow the predecessor
    if (threadIdx.x == 0) *cnt_slot = count ? __ldg(count) : batch;
  }
  __syncthreads();
  const int nb = min(batch, *cnt_slot);
  const int n_items = nb * heads;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (elect_one_sync()) {
      int t = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++t) {
        const int st = t % kApStages;
        const uint32_t ph = (t / kApStages) & 1;
        mbar_wait(empty + st, ph ^ 1);
        if (dep.wait) {   // Q, K, V^T of sequence it / heads published by the QKV GEMM
          dep_wait_geq(dep.wait + it / heads, dep.need);
          fence_proxy_async_global();
        }
        uint8_t* sb = smem + kApOffStage + st * kApStageBytes;
        mbar_expect_tx(full + st, 49152 + (mask ? 512 : 0));
        const int li = (dbg & 1) ? (int)blockIdx.x : it;
        tma_load_2d(sb, &map_q, full + st, 0, li * kAttnS);
        tma_load_2d(sb + 16384, &map_k, full + st, 0, li * kAttnS);
        tma_load_2d(sb + 32768, &map_vt, full + st, 0, li * kAttnD);
        tma_load_2d(sb + 40960, &map_vt, full + st, 64, li * kAttnD);
        if (mask) bulk_load(sb + 49152, mask + (int64_t)(it / heads) * kAttnS, 512, full + st);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    // Non-blocking scheduler: S(t) = Q K^T is issued as soon as item t's stage
    // has landed and its group's S buffer is free; O(t) = P V as soon as P(t)
    // is written and the O buffer is free.  Neither waits behind the other, so
    // a late load never holds back the PV of an item already in softmax.
    constexpr uint32_t idesc_s = idesc_bf16_f32(128, 128);
    constexpr uint32_t idesc_o = idesc_bf16_f32(128, 64);
    const int my_items = blockIdx.x < n_items ? (n_items - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    int ns = 0, no = 0;   // next item to issue S for / O for
    while (no < my_items) {
      bool done_any = false;
      if (ns < my_items) {
        const int st = ns % kApStages, gb = ns & 1;
        if (mbar_test(full + st, (ns / kApStages) & 1) && mbar_test(s_empty + gb, ((ns >> 1) & 1) ^ 1)) {
          tc_fence_after();
          if (elect_one_sync()) {
            const uint32_t sq = smem_u32(smem + kApOffStage + st * kApStageBytes);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              umma_bf16(tmem + gb * 128, sdesc_k_sw128(sq + kk * 32), sdesc_k_sw128(sq + 16384 + kk * 32),
                        idesc_s, kk != 0);
            umma_commit(s_full + gb);
          }
          __syncwarp();
          ++ns;
          done_any = true;
        }
      }
      if (no < ns) {
        const int ub = no & 1;
        const uint32_t uph = (no >> 1) & 1;
        if (mbar_test(p_full + ub, uph) && mbar_test(o_empty + ub, uph ^ 1)) {
          tc_fence_after();
          if (elect_one_sync()) {
            const uint32_t sp = smem_u32(smem + kApOffP + ub * 32768);
            const uint32_t sv = smem_u32(smem + kApOffStage + (no % kApStages) * kApStageBytes + 32768);
#pragma unroll
            for (int kb = 0; kb < 2; ++kb)
#pragma unroll
              for (int kk = 0; kk < 4; ++kk)
                umma_bf16(tmem + 256 + ub * 64, sdesc_k_sw128(sp + kb * 16384 + kk * 32),
                          sdesc_k_sw128(sv + kb * 8192 + kk * 32), idesc_o, (kb | kk) != 0);
            umma_commit(o_full + ub);
            umma_commit(empty + no % kApStages);
          }
          __syncwarp();
          ++no;
          done_any = true;
        }
      }
      if (!done_any) __nanosleep(32);
    }
  } else {
    // ------- compute groups: softmax + epilogue, thread = query row -------
    // group g = (warp - 2) / 4 owns the items t = g, g + 2, ... of this CTA:
    // softmax(t) -> [MMA: O(t)] -> epilogue(t) -> softmax(t + 2) ...; the other
    // group's softmax runs while this one waits for O(t).
    const int g = (warp - 2) >> 2;
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
    const bool leader = threadIdx.x == 64 + 128 * g;   // lane 0 of the group's first warp
    const float l2e = 1.4426950408889634f;
    uint8_t* prow = smem + kApOffP + g * 32768 + (row >> 3) * 1024 + (row & 7) * 128;
    uint8_t* orow = smem + kApOffP + g * 32768 + row * 128;   // staging tile reuses P
    int t = g;
    int prev_b = -1;   // sequence of this group's previous item, published one item late
    for (int it = blockIdx.x + g * gridDim.x; it < n_items; it += 2 * gridDim.x, t += 2) {
      const uint32_t ph = (t >> 1) & 1;
      if (t >= 2) {                        // the previous ctx store has read the P buffer
        if (leader) bulk_wait_read<0>();
        named_bar_sync(1 + g, 128);
      }
      // ---- softmax(t): the row's 128 scores in registers
      mbar_wait(s_full + g, ph);
      tc_fence_after();
      uint32_t r[4][32];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld_32x32b_x32(lane_base + g * 128 + c * 32, r[c]);
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(s_empty + g);
      float mx = -INFINITY;
      if (mask) {
        const int4* mrow = reinterpret_cast<const int4*>(smem + kApOffStage + (t % kApStages) * kApStageBytes + 49152);
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            const int4 m4 = mrow[(c * 32 + i) >> 2];   // same address in every lane: broadcast
            if (m4.x == 0) r[c][i] = __float_as_uint(-INFINITY);
            if (m4.y == 0) r[c][i + 1] = __float_as_uint(-INFINITY);
            if (m4.z == 0) r[c][i + 2] = __float_as_uint(-INFINITY);
            if (m4.w == 0) r[c][i + 3] = __float_as_uint(-INFINITY);
          }
      }
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int i = 0; i < 32; i += 2) mx = fmax3(mx, __uint_as_float(r[c][i]), __uint_as_float(r[c][i + 1]));
      const float mref = (mx == -INFINITY) ? 0.0f : mx * l2e;
      const uint64_t l2e2 = f2_pack(l2e, l2e), nm2 = f2_pack(-mref, -mref);
      uint64_t sum2 = f2_pack(0.0f, 0.0f);
      // unnormalized P row (every value <= 1) -> A operand (K-major, SW128); packed
      // fp32x2 FMA / add around the scalar MUFU ex2
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float e[8];
#pragma unroll
          for (int j = 0; j < 8; j += 2) {
            float y0, y1;
            f2_unpack(f2_fma(f2_pack(__uint_as_float(r[c][8 * q + j]), __uint_as_float(r[c][8 * q + j + 1])),
                             l2e2, nm2), y0, y1);
            e[j] = ex2_approx(y0);
            e[j + 1] = ex2_approx(y1);
            sum2 = f2_add(sum2, f2_pack(e[j], e[j + 1]));
          }
          uint4 u;
          u.x = pack_bf16(e[0], e[1]);
          u.y = pack_bf16(e[2], e[3]);
          u.z = pack_bf16(e[4], e[5]);
          u.w = pack_bf16(e[6], e[7]);
          const int chunk = (c & 1) * 4 + q;
          *reinterpret_cast<uint4*>(prow + (c >> 1) * 16384 + ((chunk ^ (row & 7)) << 4)) = u;
        }
      float s0, s1;
      f2_unpack(sum2, s0, s1);
      const float sum = s0 + s1;
      const float inv = sum > 0.0f ? 1.0f / sum : 0.0f;
      fence_proxy_async_smem();
      mbar_arrive(p_full + g);
      // ---- epilogue(t): O row / sum -> bf16 -> SW128 staging -> TMA store
      mbar_wait(o_full + g, ph);
      tc_fence_after();
      uint32_t o[2][32];
      tmem_ld_32x32b_x32(lane_base + 256 + g * 64, o[0]);
      tmem_ld_32x32b_x32(lane_base + 256 + g * 64 + 32, o[1]);
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(o_empty + g);
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const uint32_t* v = &o[c >> 2][(c & 3) * 8];
        uint4 u;
        u.x = pack_bf16(__uint_as_float(v[0]) * inv, __uint_as_float(v[1]) * inv);
        u.y = pack_bf16(__uint_as_float(v[2]) * inv, __uint_as_float(v[3]) * inv);
        u.z = pack_bf16(__uint_as_float(v[4]) * inv, __uint_as_float(v[5]) * inv);
        u.w = pack_bf16(__uint_as_float(v[6]) * inv, __uint_as_float(v[7]) * inv);
        *reinterpret_cast<uint4*>(orow + ((c ^ (row & 7)) << 4)) = u;
      }
      fence_proxy_async_smem();
      named_bar_sync(1 + g, 128);
      if (leader && !(dbg & 4)) {
        tma_store_2d(&map_o, smem + kApOffP + g * 32768, (it % heads) * kAttnD, (it / heads) * kAttnS);
        bulk_commit();
      }
      if (leader && dep.signal) {   // the previous item's ctx box has landed: publish it
        bulk_wait<1>();
        if (prev_b >= 0) {
          fence_proxy_async_global();
          dep_signal_add(dep.signal + prev_b, 1);
        }
        prev_b = it / heads;
      }
    }
    if (leader) {
      bulk_wait<0>();
      if (dep.signal && prev_b >= 0) {
        fence_proxy_async_global();
        dep_signal_add(dep.signal + prev_b, 1);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}


// ---------------------------------------------------------------------------
// attention_tp: attention_persist with the probabilities kept in tensor memory.
// The softmax writes its unnormalized bf16 P row back into the first 64 TMEM
// columns of its own S buffer (tcgen05.st) and O = P V reads A from TMEM (the
// "ts" MMA form), so P never touches shared memory: no P stores, no async-proxy
// fence, and the 64 KB of P buffers become a fourth load stage (HBM / L2
// latency: loads in flight per SM).  S(t + 2) of a group is issued only after
// O(t) (same TMEM columns; MMAs execute in issue order).
//   smem: 4 stages x (Q 16K | K 16K | V^T 16K), 2 x 16 KB ctx staging tiles,
//         4 x 512 B key-mask rows, barriers
//   TMEM: S / P buffers [0, 256) (128 columns per group), O buffers [256, 384)
__device__ unsigned long long g_attn_tl[64 * 8];   // GG_ATTN_DBG & 16 probe timeline
constexpr int kTpStageBytes = 49152;
constexpr int kTpOffStg = 4 * kTpStageBytes;              // 2 x 16 KB
constexpr int kTpOffMask = kTpOffStg + 2 * 16384;         // 4 x 512 B
constexpr int kTpOffBar = kTpOffMask + 4 * 512;
constexpr int kTpSmemNeed = kTpOffBar + 256;              // from a 1 KB-aligned base
constexpr int kTpSmem = 232448;                           // the per-CTA maximum

__global__ void __launch_bounds__(kApThreads, 1)
    attention_tp(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_k,
                 const __grid_constant__ CUtensorMap map_vt, const __grid_constant__ CUtensorMap map_o,
                 const int32_t* mask, int batch, int heads, const int32_t* count, gg_dep dep, int dbg) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t raw_u32 = smem_u32(smem_raw);
  const uint32_t pad = ((raw_u32 + 1023u) & ~1023u) - raw_u32;
  uint8_t* smem = smem_raw + pad;
  // four stages when the window's alignment leaves room, else three
  const int nst = (int)pad + kTpSmemNeed <= kTpSmem ? 4 : 3;
  if ((dbg & 8) && blockIdx.x == 0 && threadIdx.x == 0) printf("attention_tp: smem pad %u, %d stages\n", pad, nst);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (nst == 4 ? kTpOffBar : kTpOffBar - kTpStageBytes));
  uint8_t* stg0 = smem + (nst == 4 ? kTpOffStg : kTpOffStg - kTpStageBytes);
  uint8_t* mask0 = smem + (nst == 4 ? kTpOffMask : kTpOffMask - kTpStageBytes);
  uint64_t* full = bars;          // [4] stage loaded (tx bytes)
  uint64_t* empty = bars + 4;     // [4] stage free (MMA commit after O)
  uint64_t* s_full = bars + 8;    // [2] S in TMEM, per group
  uint64_t* p_full = bars + 10;   // [2] P written to TMEM by the group's 128 threads
  uint64_t* o_full = bars + 12;   // [2] O in TMEM
  uint64_t* o_empty = bars + 14;  // [2] O read by the group's 128 threads
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 16);
  int* cnt_slot = reinterpret_cast<int*>(bars + 17);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // GG_ATTN_DBG & 16: per-item timeline of CTA 0 (probe; tools/attn_probe.py)
  unsigned long long* tl = (dbg & 16) && blockIdx.x == 0 ? g_attn_tl : nullptr;
  auto now_ns = []() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
  };

  griddep_launch();
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) {
      mbar_init(full + i, 1);
      mbar_init(empty + i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(s_full + i, 1);
      mbar_init(p_full + i, 128);
      mbar_init(o_full + i, 1);
      mbar_init(o_empty + i, 128);
    }
    fence_mbar_init();
    tma_prefetch(&map_q);
    tma_prefetch(&map_k);
    tma_prefetch(&map_vt);
    tma_prefetch(&map_o);
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (dep.wait) {
    if (threadIdx.x == 0) {
      dep_wait_geq(dep.go, 1);
      *cnt_slot = count ? ld_relaxed_gpu(count) : batch;
    }
  } else {
    griddep_wait();     // Q/K/V, the mask and the count follow the predecessor
    if (threadIdx.x == 0) *cnt_slot = count ? __ldg(count) : batch;
  }
  __syncthreads();
  const int nb = min(batch, *cnt_slot);
  const int n_items = nb * heads;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (elect_one_sync()) {
      int t = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++t) {
        const int st = t % nst;
        const uint32_t ph = (t / nst) & 1;
        mbar_wait(empty + st, ph ^ 1);
        if (dep.wait) {
          dep_wait_geq(dep.wait + it / heads, dep.need);
          fence_proxy_async_global();
        }
        uint8_t* sb = smem + st * kTpStageBytes;
        if (tl) tl[t * 8 + 0] = now_ns();
        mbar_expect_tx(full + st, 49152 + (mask ? 512 : 0));
        tma_load_2d(sb, &map_q, full + st, 0, it * kAttnS);
        tma_load_2d(sb + 16384, &map_k, full + st, 0, it * kAttnS);
        tma_load_2d(sb + 32768, &map_vt, full + st, 0, it * kAttnD);
        tma_load_2d(sb + 40960, &map_vt, full + st, 64, it * kAttnD);
        if (mask) bulk_load(mask0 + st * 512, mask + (int64_t)(it / heads) * kAttnS, 512, full + st);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (non-blocking scheduler) ----------------
    constexpr uint32_t idesc_s = idesc_bf16_f32(128, 128);
    constexpr uint32_t idesc_o = idesc_bf16_f32(128, 64);
    const int my_items = blockIdx.x < n_items ? (n_items - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    int ns = 0, no = 0;   // next item to issue S for / O for
    while (no < my_items) {
      bool done_any = false;
      // S(ns) once its stage landed and O(ns - 2) (same group, same TMEM columns) is issued
      if (ns < my_items && ns < no + 2) {
        const int st = ns % nst, gb = ns & 1;
        if (mbar_test(full + st, (ns / nst) & 1)) {
          tc_fence_after();
          if (elect_one_sync()) {
            const uint32_t sq = smem_u32(smem + st * kTpStageBytes);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              umma_bf16(tmem + gb * 128, sdesc_k_sw128(sq + kk * 32), sdesc_k_sw128(sq + 16384 + kk * 32),
                        idesc_s, kk != 0);
            umma_commit(s_full + gb);
          }
          __syncwarp();
          ++ns;
          done_any = true;
        }
      }
      if (no < ns) {
        const int ub = no & 1;
        const uint32_t uph = (no >> 1) & 1;
        if (mbar_test(p_full + ub, uph) && mbar_test(o_empty + ub, uph ^ 1)) {
          tc_fence_after();
          if (elect_one_sync()) {
            const uint32_t sv = smem_u32(smem + (no % nst) * kTpStageBytes + 32768);
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)   // K = 128 keys: P columns 8 kk.., V^T key block kk / 4
              umma_bf16_ts(tmem + 256 + ub * 64, tmem + ub * 128 + kk * 8,
                           sdesc_k_sw128(sv + (kk >> 2) * 8192 + (kk & 3) * 32), idesc_o, kk != 0);
            umma_commit(o_full + ub);
            umma_commit(empty + no % nst);
          }
          __syncwarp();
          ++no;
          done_any = true;
        }
      }
      if (!done_any) __nanosleep(32);
    }
  } else {
    // ------- compute groups: softmax + epilogue, thread = query row -------
    const int g = (warp - 2) >> 2;
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
    const bool leader = threadIdx.x == 64 + 128 * g;
    const float l2e = 1.4426950408889634f;
    uint8_t* stg = stg0 + g * 16384;
    uint8_t* orow = stg + row * 128;
    int t = g;
    int prev_b = -1;
    for (int it = blockIdx.x + g * gridDim.x; it < n_items; it += 2 * gridDim.x, t += 2) {
      const uint32_t ph = (t >> 1) & 1;
      // ---- softmax(t): two passes over the row's 128 scores straight from TMEM
      // (max, then exp -> bf16 P back into TMEM), 64 / 32 scores in registers
      if (tl && (threadIdx.x & 127) == 64) tl[t * 8 + 1] = now_ns();
      mbar_wait(s_full + g, ph);
      if (tl && (threadIdx.x & 127) == 64) tl[t * 8 + 2] = now_ns();
      tc_fence_after();
      const int4* mrow = reinterpret_cast<const int4*>(mask0 + (t % nst) * 512);
      auto apply_mask = [&](uint32_t (&r)[32], int c) {
        if (!mask) return;
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          const int4 m4 = mrow[(c * 32 + i) >> 2];   // same address in every lane: broadcast
          if (m4.x == 0) r[i] = __float_as_uint(-INFINITY);
          if (m4.y == 0) r[i + 1] = __float_as_uint(-INFINITY);
          if (m4.z == 0) r[i + 2] = __float_as_uint(-INFINITY);
          if (m4.w == 0) r[i + 3] = __float_as_uint(-INFINITY);
        }
      };
      float mx = -INFINITY;
      {   // pass 1: all four 32-column loads in flight, one wait
        uint32_t r[4][32];
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_ld_32x32b_x32(lane_base + g * 128 + c * 32, r[c]);
        tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          apply_mask(r[c], c);
#pragma unroll
          for (int i = 0; i < 32; i += 2) mx = fmax3(mx, __uint_as_float(r[c][i]), __uint_as_float(r[c][i + 1]));
        }
      }
      const float mref = (mx == -INFINITY) ? 0.0f : mx * l2e;
      const uint64_t l2e2 = f2_pack(l2e, l2e), nm2 = f2_pack(-mref, -mref);
      uint64_t sum2 = f2_pack(0.0f, 0.0f);
      // pass 2: unnormalized P row (every value <= 1), bf16 pairs -> TMEM columns
      // [g*128, g*128 + 64); chunk c + 1's load is in flight while chunk c is
      // computed, and chunk c's 16 packed columns overwrite scores already read
      uint32_t r[2][32];
      tmem_ld_32x32b_x32(lane_base + g * 128, r[0]);
      tmem_ld_wait();
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (c + 1 < 4) tmem_ld_32x32b_x32(lane_base + g * 128 + (c + 1) * 32, r[(c + 1) & 1]);
        uint32_t (&rc)[32] = r[c & 1];
        apply_mask(rc, c);
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          float y0, y1;
          f2_unpack(f2_fma(f2_pack(__uint_as_float(rc[i]), __uint_as_float(rc[i + 1])), l2e2, nm2), y0, y1);
          const float e0 = ex2_approx(y0), e1 = ex2_approx(y1);
          sum2 = f2_add(sum2, f2_pack(e0, e1));
          pk[i >> 1] = pack_bf16(e0, e1);
        }
        tmem_st_32x32b_x16(lane_base + g * 128 + c * 16, pk);
        if (c + 1 < 4) tmem_ld_wait();
      }
      float s0, s1;
      f2_unpack(sum2, s0, s1);
      const float sum = s0 + s1;
      const float inv = sum > 0.0f ? 1.0f / sum : 0.0f;
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(p_full + g);
      if (tl && (threadIdx.x & 127) == 64) tl[t * 8 + 3] = now_ns();
      // ---- epilogue(t): O row / sum -> bf16 -> SW128 staging -> TMA store
      mbar_wait(o_full + g, ph);
      if (tl && (threadIdx.x & 127) == 64) tl[t * 8 + 4] = now_ns();
      tc_fence_after();
      uint32_t o[2][32];
      tmem_ld_32x32b_x32(lane_base + 256 + g * 64, o[0]);
      tmem_ld_32x32b_x32(lane_base + 256 + g * 64 + 32, o[1]);
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(o_empty + g);
      if (t >= 2) {                        // the previous ctx store has read the staging tile
        if (leader) bulk_wait_read<0>();
        named_bar_sync(1 + g, 128);
      }
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const uint32_t* v = &o[c >> 2][(c & 3) * 8];
        uint4 u;
        u.x = pack_bf16(__uint_as_float(v[0]) * inv, __uint_as_float(v[1]) * inv);
        u.y = pack_bf16(__uint_as_float(v[2]) * inv, __uint_as_float(v[3]) * inv);
        u.z = pack_bf16(__uint_as_float(v[4]) * inv, __uint_as_float(v[5]) * inv);
        u.w = pack_bf16(__uint_as_float(v[6]) * inv, __uint_as_float(v[7]) * inv);
        *reinterpret_cast<uint4*>(orow + ((c ^ (row & 7)) << 4)) = u;
      }
      fence_proxy_async_smem();
      named_bar_sync(1 + g, 128);
      if (leader) {
        if (tl) tl[t * 8 + 5] = now_ns();
        tma_store_2d(&map_o, stg, (it % heads) * kAttnD, (it / heads) * kAttnS);
        bulk_commit();
        if (dep.signal) {   // the previous item's ctx box has landed: publish it
          bulk_wait<1>();
          if (prev_b >= 0) {
            fence_proxy_async_global();
            dep_signal_add(dep.signal + prev_b, 1);
          }
          prev_b = it / heads;
        }
      }
    }
    if (leader) {
      bulk_wait<0>();
      if (dep.signal && prev_b >= 0) {
        fence_proxy_async_global();
        dep_signal_add(dep.signal + prev_b, 1);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

}  // namespace gg

using namespace gg;

static int attention_impl(const void* qkv, const int32_t* mask, void* ctx, int64_t ldc,
                          int32_t batch, int32_t heads, int32_t seq_len, const int32_t* count_dev,
                          const gg_dep* dep_in, void* stream) {
  if (!qkv || !ctx || batch <= 0 || heads <= 0) return GG_ERR_INVALID_ARGUMENT;
  gg_dep dep{nullptr, 0, nullptr, nullptr, nullptr};
  if (dep_in && (dep_in->wait || dep_in->signal)) {
    if (!dep_in->go || (dep_in->wait && dep_in->need <= 0)) return GG_ERR_INVALID_ARGUMENT;
    dep = *dep_in;
  }
  if (seq_len != kAttnS || ldc % 8 || ldc < (int64_t)heads * kAttnD) return GG_ERR_UNSUPPORTED;
  const int64_t plane = (int64_t)batch * heads * seq_len * kAttnD;
  const __nv_bfloat16* base = reinterpret_cast<const __nv_bfloat16*>(qkv);
  CUtensorMap mq, mk, mv;
  const int64_t rows = (int64_t)batch * heads * seq_len;
  int rc = make_map_2d(&mq, base, rows, kAttnD, kAttnD, 128);
  if (!rc) rc = make_map_2d(&mk, base + plane, rows, kAttnD, kAttnD, 128);
  if (!rc) rc = make_map_2d(&mv, base + 2 * plane, (int64_t)batch * heads * kAttnD, seq_len, seq_len, 64);
  if (rc) return rc;
  static const bool simple = getenv("GG_ATTN_SIMPLE") != nullptr;
  // GG_ATTN_DBG (probe switches, tools/attn_probe.py; never set in production):
  // 1 = every CTA reloads its first item (L2-resident loads), 2 = no exp in the
  // softmax, 4 = no ctx stores
  static const int dbg = getenv("GG_ATTN_DBG") ? atoi(getenv("GG_ATTN_DBG")) : 0;
  static const bool smem_p = getenv("GG_ATTN_SMEM_P") != nullptr;   // A/B: P through shared memory
  if (!simple && !smem_p && !(dbg & 7)) {
    CUtensorMap mo;
    if (int rc2 = make_map_2d(&mo, ctx, (int64_t)batch * seq_len, (int64_t)heads * kAttnD, ldc, 128))
      return rc2;
    static bool tattr = false;
    if (!tattr) {
      if (cudaFuncSetAttribute(attention_tp, cudaFuncAttributeMaxDynamicSharedMemorySize, kTpSmem) !=
          cudaSuccess)
        return GG_ERR_CUDA;
      tattr = true;
    }
    const int grid = (int)std::min<int64_t>((int64_t)batch * heads, num_sms());
    if (launch_pdl(attention_tp, dim3(grid), dim3(kApThreads), kTpSmem, gg_stream(stream), mq, mk, mv, mo,
                   mask, batch, heads, count_dev, dep, dbg) != cudaSuccess)
      return GG_ERR_CUDA;
    GG_LAUNCH_OK();
    if (dbg & 16) {
      unsigned long long h[64 * 8];
      cudaDeviceSynchronize();
      cudaMemcpyFromSymbol(h, g_attn_tl, sizeof(h));
      const unsigned long long t0 = h[0];
      for (int t = 0; t < 12; ++t)
        fprintf(stderr, "attn item %2d: load issued %7.2f  S wait %7.2f -> %7.2f  P done %7.2f  O ready %7.2f  "
                "store %7.2f us\n", t, (h[t * 8] - t0) * 1e-3, (h[t * 8 + 1] - t0) * 1e-3,
                (h[t * 8 + 2] - t0) * 1e-3, (h[t * 8 + 3] - t0) * 1e-3, (h[t * 8 + 4] - t0) * 1e-3,
                (h[t * 8 + 5] - t0) * 1e-3);
    }
    return GG_OK;
  }
  if (!simple) {
    CUtensorMap mo;
    if (int rc2 = make_map_2d(&mo, ctx, (int64_t)batch * seq_len, (int64_t)heads * kAttnD, ldc, 128))
      return rc2;
    static bool pattr = false;
    if (!pattr) {
      if (cudaFuncSetAttribute(attention_persist, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               kApSmem) != cudaSuccess)
        return GG_ERR_CUDA;
      pattr = true;
    }
    const int grid = (int)std::min<int64_t>((int64_t)batch * heads, num_sms());
    if (launch_pdl(attention_persist, dim3(grid), dim3(kApThreads), kApSmem, gg_stream(stream), mq, mk,
                   mv, mo, mask, batch, heads, count_dev, dbg, dep) != cudaSuccess)
      return GG_ERR_CUDA;
    GG_LAUNCH_OK();
    return GG_OK;
  }
  if (dep.wait || dep.signal) return GG_ERR_UNSUPPORTED;   // the per-item kernel has no deps
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(attention_tcgen05, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             kAttnSmem) != cudaSuccess)
      return GG_ERR_CUDA;
    attr = true;
  }
  if (launch_pdl(attention_tcgen05, dim3(batch * heads), dim3(kAttnThreads), kAttnSmem, gg_stream(stream),
                 mq, mk, mv, mask, reinterpret_cast<__nv_bfloat16*>(ctx), ldc, heads, count_dev) != cudaSuccess)
    return GG_ERR_CUDA;
  GG_LAUNCH_OK();
  return GG_OK;
}

extern "C" int gg_attention(const void* qkv, const int32_t* mask, void* ctx, int64_t ldc,
                            int32_t batch, int32_t heads, int32_t seq_len,
                            const int32_t* count_dev, void* stream) {
  return attention_impl(qkv, mask, ctx, ldc, batch, heads, seq_len, count_dev, nullptr, stream);
}

extern "C" int gg_attention_dep(const void* qkv, const int32_t* mask, void* ctx, int64_t ldc,
                                int32_t batch, int32_t heads, int32_t seq_len,
                                const int32_t* count_dev, const gg_dep* dep, void* stream) {
  if (!dep) return GG_ERR_INVALID_ARGUMENT;
  return attention_impl(qkv, mask, ctx, ldc, batch, heads, seq_len, count_dev, dep, stream);
}
