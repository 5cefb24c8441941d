// gg_tc.cuh — sm_100a tensor-core plumbing: mbarriers, TMA, tcgen05 (UMMA/TMEM).
// Inline PTX only; descriptor bit layouts follow the PTX ISA for tcgen05
// (shared-memory matrix descriptor and kind::f16 instruction descriptor).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace gg {
namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---- mbarrier ---------------------------------------------------------------
// Round a dynamic-smem pointer up to 1 KB (SWIZZLE_128B atoms) while staying in
// the shared address space: offsetting the array itself keeps LDS / STS; a round
// trip through an integer address makes every access through the result generic.
__device__ __forceinline__ uint8_t* smem_align1k(uint8_t* base) {
  const uint32_t a = smem_u32(base);
  return base + (((a + 1023u) & ~1023u) - a);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Non-blocking probe: has the phase with this parity completed?
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.b32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// Wait with a hardware suspend hint: the thread sleeps until the phase completes
// (or the hint elapses) instead of spinning.  For the producer and epilogue warps,
// whose hot try_wait loops otherwise take issue slots from the single MMA-issuing
// thread on the same SM sub-partition.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAITS_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAITS_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(20000u)
      : "memory");
}

// One lane of a converged warp (PTX elect.sync).  The MMA-issuing warp runs its
// loop warp-uniformly and issues each batch of tcgen05.mma / commit inside
// `if (elect_one_sync())`: ptxas then emits the UTCHMMAs back to back from
// uniform registers.  Issuing from a `lane == 0` branch instead wraps every
// UTCHMMA in an ELECT / BRA.U.ANY loop (~9 dependent instructions per MMA),
// which at N = 64 (32-48 tensor cycles per MMA) made the stem and layer-1 convs
// issue-bound at ~110 cycles per MMA.
__device__ __forceinline__ bool elect_one_sync() {
  uint32_t pred = 0;
  asm volatile(
      "{\n.reg .b32 r;\n.reg .pred P;\nelect.sync r|P, 0xffffffff;\nselp.b32 %0, 1, 0, P;\n}\n"
      : "=r"(pred));
  return pred != 0;
}

// ---- TMA ----------------------------------------------------------------------
__device__ __forceinline__ void tma_prefetch(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int32_t x, int32_t y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(x), "r"(y)
      : "memory");
}
// 1-D bulk copy global -> shared (bytes % 16 == 0, both addresses 16-B aligned).
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int32_t x, int32_t y, int32_t z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z)
      : "memory");
}

// ---- tcgen05 ------------------------------------------------------------------
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// D[tmem] (+)= A[smem] * B[smem]^T, bf16 inputs, fp32 accumulate, cta_group::1.
__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Arrive on an mbarrier when all previously issued tcgen05.mma of this thread complete.
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

// 32 lanes x 32 consecutive fp32 columns per warp (lane quarter = warp % 4).
__device__ __forceinline__ void tmem_ld_32x32b_x32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
// 32 lanes x 32 consecutive 32-bit columns from registers into TMEM.
__device__ __forceinline__ void tmem_st_32x32b_x32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]),
      "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]),
      "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]),
      "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tmem_st_32x32b_x16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
// D[tmem] (+)= A[tmem] . B[smem]^T: the A operand (M lanes x K, two bf16 per
// 32-bit column, row = lane) read from tensor memory instead of shared memory.
__device__ __forceinline__ void umma_bf16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                             uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Shared-memory matrix descriptor, K-major, 128-byte swizzle: 8-row x 128 B
// atoms, SBO = 1024 B between 8-row groups, LBO unused (1), version 1 (sm_100).
__device__ __forceinline__ uint64_t sdesc_k_sw128(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;                 // LBO (ignored for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;       // SBO
  d |= (uint64_t)1 << 46;                 // descriptor version (Blackwell)
  // base offset (bits 49-51) stays 0: the swizzle XOR is applied to the
  // absolute smem address bits [7:9], so a start shifted by whole 128-B rows
  // inside an atom addresses correctly (verified by tests/test_conv_span_gpu.py)
  d |= (uint64_t)2 << 61;                 // SWIZZLE_128B
  return d;
}

// K-major, 32-byte swizzle (rows of 16 bf16 = one UMMA K step), 8-row atoms of
// 256 B stacked densely along M/N.  Used for 16-channel im2col tiles.
__device__ __forceinline__ uint64_t sdesc_k_sw32(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(256 >> 4) << 32;        // SBO: 8 rows x 32 B
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)6 << 61;                 // SWIZZLE_32B
  return d;
}

// kind::f16 instruction descriptor: bf16 A/B, fp32 D, both K-major.
__host__ __device__ constexpr uint32_t idesc_bf16_f32(int M, int N) {
  return (1u << 4)                 // D format f32
         | (1u << 7)               // A format bf16
         | (1u << 10)              // B format bf16
         | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// Exact-erf GELU, x * Phi(x), for the GEMM epilogue at tensor-core pace.
// With a = min(|x|, 5.75): Phi(-a) = erfc(a / sqrt 2) / 2 = 2^q(a) / 2, q a
// degree-8 Chebyshev fit of log2 erfc(a / sqrt 2) on [0, 5.75]; then
// gelu(x) = x - x Phi(-x) for x >= 0 and x Phi(x) below.  One MUFU ex2 and nine
// FMAs instead of erff's branchy ~40 instructions (the epilogue issue rate
// bounded the FFN-up GEMM); |gelu_erf - exact| <= 4.2e-7 over all fp32 x
// (tools/fit_gelu.py), 10^4 below the bf16 rounding of the stored output.
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float tanh_approx(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
#ifdef GG_GELU_TANH
__device__ __forceinline__ float gelu_erf(float x) {
  const float u = x * fmaf(0.0356774081f, x * x, 0.7978845608f);
  const float hx = 0.5f * x;
  return fmaf(hx, tanh_approx(u), hx);
}
#else
__device__ __forceinline__ float gelu_erf(float x) {
  const float a = fminf(fabsf(x), 5.75f);
  float q = -3.1597807037542225e-08f;
  q = fmaf(q, a, -1.2583882380567957e-06f);
  q = fmaf(q, a, 5.780859646620229e-05f);
  q = fmaf(q, a, -0.0009210868738591671f);
  q = fmaf(q, a, 0.008511481806635857f);
  q = fmaf(q, a, -0.05401911586523056f);
  q = fmaf(q, a, -0.45836740732192993f);
  q = fmaf(q, a, -1.1513043642044067f);
  q = fmaf(q, a, 1.1678074770316016e-05f);
  const float e = 0.5f * x * ex2_approx(q);
  return x >= 0.0f ? x - e : e;
}
#endif

// ---- packed fp32x2 arithmetic (sm_100: FFMA2 / FMUL2 / FADD2, two lanes of
// IEEE fp32 per instruction; identical rounding to the scalar ops) ----------
__device__ __forceinline__ uint64_t f2_pack(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void f2_unpack(uint64_t v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ uint64_t f2_fma(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t f2_mul(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t f2_add(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

// three-input max (FMNMX3)
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

// GELU on a pair with packed arithmetic (the FFN-up epilogue bounds that GEMM).
// With a = min(|x|, 5.75) and d = a Phi(-a) = a 2^(q(a) - 1), q a degree-6 fit
// of log2 erfc(a / sqrt 2) on [0, 5.75] (the -1 folded into the constant term):
//   gelu(x) = x Phi(x) = max(x, 0) - d
// (x >= 0: x - x Phi(-x); x < 0: x Phi(-|x|) = -d).  14 instructions per pair
// (2 clamps, 6 FFMA2, 2 MUFU ex2, FMUL2, 2 relu, FADD2); |error| <= 4.7e-6 over
// all fp32 x (tools/fit_gelu.py), 1/27 of the bf16 half-ulp the output is
// rounded to.  The scalar gelu_erf above keeps the degree-8 fit.
__device__ __forceinline__ void gelu_erf2(float& x0, float& x1) {
#ifdef GG_GELU_TANH
  x0 = gelu_erf(x0);
  x1 = gelu_erf(x1);
#else
  const uint64_t a = f2_pack(fminf(fabsf(x0), 5.75f), fminf(fabsf(x1), 5.75f));
  uint64_t q = f2_fma(f2_pack(2.4683062292751856e-05f, 2.4683062292751856e-05f), a,
                      f2_pack(-0.0006366565939970315f, -0.0006366565939970315f));
  q = f2_fma(q, a, f2_pack(0.007334418594837189f, 0.007334418594837189f));
  q = f2_fma(q, a, f2_pack(-0.05150618776679039f, -0.05150618776679039f));
  q = f2_fma(q, a, f2_pack(-0.46100395917892456f, -0.46100395917892456f));
  q = f2_fma(q, a, f2_pack(-1.1501705646514893f, -1.1501705646514893f));
  q = f2_fma(q, a, f2_pack(-1.0001055002212524f, -1.0001055002212524f));
  float q0, q1;
  f2_unpack(q, q0, q1);
  const uint64_t d = f2_mul(a, f2_pack(ex2_approx(q0), ex2_approx(q1)));
  f2_unpack(f2_add(f2_pack(fmaxf(x0, 0.0f), fmaxf(x1, 0.0f)), f2_mul(d, f2_pack(-1.0f, -1.0f))), x0, x1);
#endif
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

}  // namespace tc
}  // namespace gg

// ---- CTA pairs (cluster of 2, cta_group::2) -------------------------------------
namespace gg {
namespace tc {
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// shared::cluster address of the same shared variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_shared(uint32_t smem_addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// arrive on an mbarrier given by its shared::cluster address (possibly the peer CTA's)
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}
// mbarrier wait with cluster-scope acquire (the phase was completed by a remote
// release.cluster arrive that published data written into this CTA's smem)
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAITC_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAITC_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// relaxed arrives: signal progress without waiting for the thread's outstanding
// memory operations (ring-slot releases after the value was consumed)
__device__ __forceinline__ void mbar_arrive_relaxed(uint64_t* bar) {
  asm volatile("mbarrier.arrive.relaxed.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster_relaxed(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void st_shared_cluster_s32(uint32_t cluster_addr, int v) {
  asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(cluster_addr), "r"(v) : "memory");
}
// TMA tile load into this CTA's smem, completing bytes on an mbarrier that may
// live in the peer CTA of the pair (the leader's full barrier).
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map,
                                                 uint32_t bar_cluster, int32_t x, int32_t y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(bar_cluster), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void tmem_alloc_pair(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}
// D[tmem of both CTAs] (+)= A (M = 256: 128 rows in each CTA's smem) * B^T (N split
// in halves across the two CTAs' smem); issued by the leader CTA only.
__device__ __forceinline__ void umma_bf16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                               uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// arrive on the mbarrier at the same smem offset in every CTA of `mask` when the
// leader's previously issued pair MMAs complete
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"(mask)
      : "memory");
}
}  // namespace tc
}  // namespace gg

// ---- TMA stores (smem -> global, bulk-group completion) -------------------------
namespace gg {
namespace tc {
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int32_t x, int32_t y) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(map),
               "r"(smem_u32(src)), "r"(x), "r"(y)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
// generic-proxy smem writes -> visible to the async proxy (TMA store source)
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
}  // namespace tc
}  // namespace gg

// ---- coalesced row-chunk epilogue through a per-warp smem tile ------------------
// A TMEM accumulator load gives lane r the 32 columns of row r, so direct global
// accesses touch 32 rows (32 L1 wavefronts) per instruction.  These helpers move a
// warp's 32 rows x 32 bf16 columns (64 B per row) through a 2 KB smem tile laid out
// with the 64-byte swizzle (16-B chunk q of row r at q ^ ((r >> 1) & 3): conflict-
// free both for row-per-lane and for 4-lanes-per-row access), so each global
// instruction covers 8 rows x 64 contiguous bytes.  `off` is this lane's element
// offset of (its row, first column); rows with ok == false are skipped.
namespace gg {
namespace tc {
template <typename T>   // any 2-byte element type (bf16 / fp16)
__device__ __forceinline__ void warp_rows_load(uint8_t* buf, const T* base, int64_t off, bool ok,
                                               int lane, uint4 (&row)[4]) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int rr = j * 8 + (lane >> 2), piece = lane & 3;
    const int64_t o = __shfl_sync(0xffffffffu, off, rr);
    const bool k = __shfl_sync(0xffffffffu, ok, rr);
    uint4 u = make_uint4(0, 0, 0, 0);
    if (k) u = __ldg(reinterpret_cast<const uint4*>(base + o) + piece);
    *reinterpret_cast<uint4*>(buf + rr * 64 + ((piece ^ ((rr >> 1) & 3)) << 4)) = u;
  }
  __syncwarp();
  const int sw = (lane >> 1) & 3;
#pragma unroll
  for (int q = 0; q < 4; ++q) row[q] = *reinterpret_cast<const uint4*>(buf + lane * 64 + ((q ^ sw) << 4));
  __syncwarp();
}
// L2 eviction-priority policies (createpolicy): keep a producer's output for the
// very next kernel, stream a consumer's single-use reads
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void st_global_v4_hint(void* ptr, uint4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(ptr), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w), "l"(pol)
               : "memory");
}
__device__ __forceinline__ uint4 ld_global_nc_v4_hint(const void* ptr, uint64_t pol) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(ptr), "l"(pol));
  return v;
}

template <bool KEEP_L2 = false, typename T = __nv_bfloat16>
__device__ __forceinline__ void warp_rows_store(uint8_t* buf, T* base, int64_t off, bool ok, int lane,
                                                const uint4 (&row)[4]) {
  const int sw = (lane >> 1) & 3;
#pragma unroll
  for (int q = 0; q < 4; ++q) *reinterpret_cast<uint4*>(buf + lane * 64 + ((q ^ sw) << 4)) = row[q];
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int rr = j * 8 + (lane >> 2), piece = lane & 3;
    const int64_t o = __shfl_sync(0xffffffffu, off, rr);
    const bool k = __shfl_sync(0xffffffffu, ok, rr);
    const uint4 u = *reinterpret_cast<const uint4*>(buf + rr * 64 + ((piece ^ ((rr >> 1) & 3)) << 4));
    if (k) {
      if constexpr (KEEP_L2) st_global_v4_hint(reinterpret_cast<uint4*>(base + o) + piece, u, l2_policy_evict_last());
      else reinterpret_cast<uint4*>(base + o)[piece] = u;
    }
  }
  __syncwarp();
}
}  // namespace tc
}  // namespace gg
