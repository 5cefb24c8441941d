// mma_bench.cu — microbenchmark of back-to-back tcgen05.mma issue from one
// thread: cycles per MMA vs N and the A-operand start alignment.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/_mma_bench tools/mma_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "../paper_2601_04250_b200/csrc/gg_tc.cuh"

using namespace gg::tc;

// variant 0: A at the 1024-aligned stage base (+kk*32), like a GEMM
// variant 1: A start shifted by (i % 9) * 128 B rows (the span conv pattern)
// variant 2: A start shifted by whole atoms (i % 9) * 1024 B
// variant 3: like 0 but the accumulate flag / addresses from a lane-0-only branch
template <int N>
__global__ void __launch_bounds__(128, 1) mma_loop(int variant, int iters, long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* a = smem;                 // 48 KB
  uint8_t* b = smem + 48 * 1024;     // N x 128 B (or 16 taps x N x 32 B)
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < (48 * 1024 + N * 512) / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if ((threadIdx.x >> 5) == 0) tmem_alloc(&tslot, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 32) {
    constexpr uint32_t idesc = idesc_bf16_f32(128, N);
    const uint32_t sa = smem_u32(a), sb = smem_u32(b);
    long long t0 = clock64();
    if (variant == 5 || variant == 6) {   // SW32 (16-channel rows): the stem's operand layout
      const uint64_t a0 = sdesc_k_sw32(sa), b0 = sdesc_k_sw32(sb);
      umma_bf16(tmem, a0, b0, idesc, 0);
      for (int i = 0; i < iters / 16; ++i) {
#pragma unroll
        for (int tap = 0; tap < 16; ++tap) {
          const uint64_t ao = (uint64_t)((variant == 6 ? ((tap / 4) * 115 + tap % 4) * 32 : 0) >> 4);
          umma_bf16(tmem, a0 + ao, b0 + (uint64_t)(tap * (N * 32 / 16)), idesc, 1);
        }
      }
      umma_commit(&bar);
      mbar_wait(&bar, 0);
      long long t1 = clock64();
      if (blockIdx.x == 0) out[0] = t1 - t0;
      iters = 0;
    }
    if (variant == 3 || variant == 4) {   // lean issue: descriptors = base + constant offsets, unrolled
      const uint64_t a0 = sdesc_k_sw128(sa), b0 = sdesc_k_sw128(sb);
      umma_bf16(tmem, a0, b0, idesc, 0);
      for (int i = 0; i < iters / 36; ++i) {
#pragma unroll
        for (int tap = 0; tap < 9; ++tap) {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t ao = (uint64_t)(((variant == 4 ? tap * 128 : 0) + kk * 32) >> 4);
            umma_bf16(tmem, a0 + ao, b0 + (uint64_t)((kk * 32) >> 4), idesc, 1);
          }
        }
      }
      umma_commit(&bar);
      mbar_wait(&bar, 0);
      long long t1 = clock64();
      if (blockIdx.x == 0) out[0] = t1 - t0;
      iters = 0;
    }
    for (int i = 0; i < iters; ++i) {
      const int kk = i & 3;
      uint32_t aa = sa + kk * 32;
      if (variant == 1) aa += (uint32_t)(i % 9) * 128u;
      if (variant == 2) aa += (uint32_t)(i % 9) * 1024u;
      umma_bf16(tmem, sdesc_k_sw128(aa), sdesc_k_sw128(sb + kk * 32), idesc, i > 0);
    }
    if (variant < 3 && iters > 0) {
      umma_commit(&bar);
      mbar_wait(&bar, 0);
      long long t1 = clock64();
      if (blockIdx.x == 0) out[0] = t1 - t0;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if ((threadIdx.x >> 5) == 0) tmem_dealloc(tmem, 512);
}

template <int N>
void run(long long* d_out) {
  const int smem = 48 * 1024 + N * 512 + 2048;
  cudaFuncSetAttribute(mma_loop<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 4096;
  for (int v = 0; v < 7; ++v) {
    mma_loop<N><<<148, 128, smem>>>(v, iters, d_out);
    mma_loop<N><<<148, 128, smem>>>(v, iters, d_out);
    long long h = 0;
    cudaMemcpy(&h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
    cudaError_t e = cudaGetLastError();
    const double nm = v >= 5 ? (double)(iters / 16 * 16 + 1) : v >= 3 ? (double)(iters / 36 * 36 + 1) : (double)iters;
    printf("N=%3d variant=%d: %.1f cycles/MMA (ideal %d)  %s\n", N, v, (double)h / nm, 128 * N / 256,
           e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
}

int main() {
  long long* d_out;
  cudaMalloc(&d_out, 64);
  run<64>(d_out);
  run<128>(d_out);
  run<256>(d_out);
  return 0;
}
