// gg_streamk.cuh — stream-K work distribution for the persistent tcgen05 GEMM /
// implicit-GEMM conv kernels.
//
// Data-parallel persistent kernels give every CTA whole output tiles; when the
// tile count is not a multiple of the SM count the last wave runs partly empty
// (DistilBERT's N = 768 GEMMs: 384 tiles on 148 SMs = 2.59 waves, 86 %
// efficiency; ResNet layer 4: 100 tiles, 68 %).  Stream-K instead splits the
// flattened (tile, k-block) iteration space evenly: CTA c owns iterations
// [c*T/G, (c+1)*T/G), T = tiles * k-blocks, so every CTA does the same MMA work.
// A tile cut between CTAs is reduced through a global fp32 workspace:
//
//   * each epilogue warp owns a 32-row region of the tile and arrives on a
//     per-(tile, region) counter when its accumulator is ready;
//   * every arriver but the last writes its partial region to its CTA's slot
//     (slot 0 = the CTA's first work item, slot 1 = its last), fences, and
//     bumps a per-(tile, region) "ready" counter;
//   * the last arriver waits for ready == segments - 1 (the others are already
//     past their MMAs, so the wait is the length of a store), sums all segments
//     in k order (its own in place: deterministic for any arrival order), runs
//     the ordinary fused epilogue and resets both counters for the next launch.
//
// The workspace is per device and owned by the library (gg_streamk_reserve);
// like the models' activation buffers it serves one stream at a time.
#pragma once
#include <stdint.h>

namespace gg {

struct StreamK {
  float* ws;   // [G][2 slots][regions][32 lanes x region columns], column-major per region
  int* cnt;    // [tiles][regions][2]: arrivals, ready
  int enabled;
};

struct SkWork {
  int tile, kb0, kb1;
};

// Iterates a CTA's work items: whole tiles strided by the grid (data-parallel)
// or its contiguous stream-K range of (tile, k-block) iterations.
struct SkSched {
  int64_t pos, end, T;
  int nkb, G, sk;
  __device__ __forceinline__ SkSched(int stream_k, int num_tiles, int nkb_, int cta, int grid)
      : nkb(nkb_), G(grid), sk(stream_k) {
    T = (int64_t)num_tiles * nkb_;
    if (sk) {
      pos = (int64_t)cta * T / grid;
      end = (int64_t)(cta + 1) * T / grid;
    } else {
      pos = cta;
      end = num_tiles;
    }
  }
  __device__ __forceinline__ bool next(SkWork& w) {
    if (pos >= end) return false;
    if (!sk) {
      w.tile = (int)pos;
      w.kb0 = 0;
      w.kb1 = nkb;
      pos += G;
      return true;
    }
    w.tile = (int)(pos / nkb);
    w.kb0 = (int)(pos - (int64_t)w.tile * nkb);
    const int64_t left = end - pos;
    w.kb1 = left < nkb - w.kb0 ? w.kb0 + (int)left : nkb;
    pos += w.kb1 - w.kb0;
    return true;
  }
  // CTA whose range contains iteration p
  __device__ __forceinline__ int cta_of(int64_t p) const { return (int)(((p + 1) * G - 1) / T); }
  __device__ __forceinline__ int64_t start_of(int c) const { return (int64_t)c * T / G; }
};

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Per-warp fixup for a tile cut between CTAs (called by every epilogue warp for
// its region of a partial work item).  Returns true when this warp is the last
// arriver and must run the epilogue; `fx` then names the tile's segments (the
// CTAs c_first..c_last) for sk_sum.  Non-last arrivers store their region here
// (from TMEM through `load32`, a functor that fills 32 fp32 accumulator columns).
struct SkFix {
  int c_first, c_last, me;
};

template <int RC, typename Load32>
__device__ __forceinline__ bool sk_arrive(const StreamK& sk, const SkSched& sc, const SkWork& w,
                                          int region, int regions, int lane, SkFix& fx,
                                          Load32&& load32) {
  fx.c_first = sc.cta_of((int64_t)w.tile * sc.nkb);
  fx.c_last = sc.cta_of((int64_t)w.tile * sc.nkb + sc.nkb - 1);
  fx.me = blockIdx.x;
  const int nseg = fx.c_last - fx.c_first + 1;
  int* cnt = sk.cnt + ((int64_t)w.tile * regions + region) * 2;
  int arrive = 0;
  if (lane == 0) arrive = atomicAdd(cnt, 1);
  arrive = __shfl_sync(0xffffffffu, arrive, 0);
  if (arrive < nseg - 1) {
    const int slot = (w.tile == (int)(sc.start_of(fx.me) / sc.nkb)) ? 0 : 1;
    float* dst = sk.ws + (((int64_t)fx.me * 2 + slot) * regions + region) * (32 * RC);
#pragma unroll 1
    for (int c = 0; c < RC; c += 32) {
      float v[32];
      load32(c, v);
#pragma unroll
      for (int i = 0; i < 32; ++i) __stcg(dst + (c + i) * 32 + lane, v[i]);
    }
    __threadfence();
    __syncwarp();
    if (lane == 0) atomicAdd(cnt + 1, 1);
    return false;
  }
  while (ld_acquire(cnt + 1) < nseg - 1) __nanosleep(32);
  __syncwarp();
  if (lane == 0) {   // reset for the next launch (stream-ordered)
    cnt[0] = 0;
    cnt[1] = 0;
  }
  return true;
}

// v[0..31] (this CTA's accumulator columns c..c+31) := sum over the tile's
// segments in k order, reading the other CTAs' partial slots.
template <int RC>
__device__ __forceinline__ void sk_sum(const StreamK& sk, const SkSched& sc, const SkWork& w,
                                       int region, int regions, int lane, const SkFix& fx, int c,
                                       float (&v)[32]) {
  float acc[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) acc[i] = 0.0f;
  for (int seg = fx.c_first; seg <= fx.c_last; ++seg) {
    if (seg == fx.me) {
#pragma unroll
      for (int i = 0; i < 32; ++i) acc[i] += v[i];
    } else {
      const int slot = (w.tile == (int)(sc.start_of(seg) / sc.nkb)) ? 0 : 1;
      const float* src = sk.ws + (((int64_t)seg * 2 + slot) * regions + region) * (32 * RC);
#pragma unroll
      for (int i = 0; i < 32; ++i) acc[i] += __ldcg(src + (c + i) * 32 + lane);
    }
  }
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = acc[i];
}

}  // namespace gg

// Host side (gg_gemm.cu): the per-device workspace.
namespace gg {
// Returns the workspace of the current device, allocating it when possible
// (not while `stream` is being captured).  ok = false -> run data-parallel.
StreamK streamk_workspace(cudaStream_t stream, int64_t ws_floats, int64_t counters, bool& ok);
bool streamk_wanted(int64_t tiles, int64_t nkb, int sms);
}
