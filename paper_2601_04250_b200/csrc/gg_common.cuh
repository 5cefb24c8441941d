// gg_common.cuh — shared helpers for the greengate B200 kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/greengate_b200.h"
#include "../../include/greengate_b200_forward.h"

#define GG_CUDA_OK(expr)                                   \
  do {                                                     \
    cudaError_t _e = (expr);                               \
    if (_e != cudaSuccess) return GG_ERR_CUDA;             \
  } while (0)

#define GG_LAUNCH_OK()                                     \
  do {                                                     \
    cudaError_t _e = cudaGetLastError();                   \
    if (_e != cudaSuccess) return GG_ERR_CUDA;             \
  } while (0)

static inline cudaStream_t gg_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Programmatic dependent launch (see launch_pdl in gg_kernels.h): wait for the
// stream predecessor's completion + memory flush / let the successor's CTAs start.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" :::); }

// Tile-level dependencies between consecutive kernels (gg_dep): per-unit
// counters in global memory, released by the producer after its outputs are
// complete, acquired by the consumer before it reads them.
__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_relaxed_gpu(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void dep_wait_geq(const int* p, int need) {
  while (ld_acquire_gpu(p) < need) __nanosleep(100);
}
__device__ __forceinline__ void dep_signal_add(int* p, int v) {
  asm volatile("fence.acq_rel.gpu;\n\tred.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void dep_signal_add_nofence(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void dep_set(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// completed bulk (TMA) writes / generic acquires <-> async-proxy accesses of global memory
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// Every fp64 operation of the controller goes through these so the rounding is
// exactly CPython's (one IEEE rounding per binary op, no FMA contraction).
__device__ __forceinline__ double f64_add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double f64_sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double f64_mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double f64_div(double a, double b) { return __ddiv_rn(a, b); }

// CPython 3.12 builtin sum() over floats: Neumaier compensation
// (Objects/bltinmodule.c builtin_sum_impl; used by controller.py:132, 141).
struct NeumaierSum {
  double s = 0.0, c = 0.0;
  __device__ __forceinline__ void add(double x) {
    // both compensation candidates are computed and one is selected (no
    // divergence, and only `s` is on the loop-carried critical path)
    const double t = f64_add(s, x);
    const double big_s = f64_add(f64_sub(s, t), x);
    const double big_x = f64_add(f64_sub(x, t), s);
    c = f64_add(c, fabs(s) >= fabs(x) ? big_s : big_x);
    s = t;
  }
  __device__ __forceinline__ double result() const {
    return (c != 0.0 && isfinite(c)) ? f64_add(s, c) : s;
  }
};

// min(1.0, max(0.0, v)) with Python's first-argument-wins ties.
__device__ __forceinline__ double clamp01(double v) {
  v = (v > 0.0) ? v : 0.0;
  return (v < 1.0) ? v : 1.0;
}

// NormalizerChannel.observe / normalize (controller.py:164-180).
__device__ __forceinline__ void ch_observe(gg_channel& c, double raw) {
  if (!c.seen || raw < c.lo) c.lo = raw;
  if (!c.seen || raw > c.hi) c.hi = raw;
  c.seen = 1;
}
__device__ __forceinline__ double ch_normalize(gg_channel& c, double raw) {
  ch_observe(c, raw);
  if (c.hi <= c.lo) return 0.0;
  return clamp01(f64_div(f64_sub(raw, c.lo), f64_sub(c.hi, c.lo)));
}
