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
__device__ int g_zero = 0;

template <int N>
__global__ void __launch_bounds__(128, 1) mma_loop(int variant, int iters, long long* out,
                                                   const uint8_t* gsrc, int copy_bytes) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* a = smem;                 // 48 KB
  uint8_t* b = smem + 48 * 1024;     // N x 128 B (or 16 taps x N x 32 B)
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < (48 * 1024 + N * 512) / 4; i += blockDim.x) {
    // random bf16 pairs in [-1, 1) (data-dependent tensor power) unless g_zero
    uint32_t h = (uint32_t)i * 2654435761u ^ 0x9e3779b9u;
    h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
    const uint32_t lo = 0x3c00u | (h & 0x7fu) | ((h & 0x100u) << 7);           // +-[0.0078, 0.0156)*...
    const uint32_t hi = 0x3f00u | ((h >> 9) & 0x7fu) | (((h >> 16) & 1u) << 15);  // +-[0.5, 1)
    reinterpret_cast<uint32_t*>(smem)[i] = g_zero ? 0u : (lo | (hi << 16));
  }
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
  __shared__ uint64_t cbar[2];
  if (variant >= 10 && threadIdx.x == 64) {   // concurrent smem writes: 15 KB bulk copies, 2 in flight
    uint8_t* ring = smem + 48 * 1024 + N * 512 + 1024;
    mbar_init(&cbar[0], 1);
    mbar_init(&cbar[1], 1);
    fence_mbar_init();
    const int n = copy_bytes > 0 ? 400 : 0;
    for (int i = 0; i < n; ++i) {
      const int s = i & 1;
      if (i >= 2) mbar_wait(&cbar[s], ((i - 2) >> 1) & 1);
      mbar_expect_tx(&cbar[s], copy_bytes);
      bulk_load(ring + s * 16384, gsrc + (size_t)(blockIdx.x * 400 + i) % 4096 * 16384, copy_bytes, &cbar[s]);
    }
    if (n >= 2) { mbar_wait(&cbar[0], ((n - 2) >> 1) & 1); mbar_wait(&cbar[1], ((n - 1) >> 1) & 1); }
  }
  if (threadIdx.x == 32) {
    constexpr uint32_t idesc = idesc_bf16_f32(128, N);
    const uint32_t sa = smem_u32(a), sb = smem_u32(b);
    long long t0 = clock64();
    if (variant >= 10) {   // variant 9 + bulk copies (warp 2, below) streaming into a separate smem ring
      variant = 9;
    }
    if (variant >= 7) {   // the stem's per-tile pattern: 16 SW32 MMAs into one of 4 accumulators, then commits
      __shared__ uint64_t bars[8];
      if (true) {
        for (int i = 0; i < 8; ++i) mbar_init(&bars[i], 1);
        fence_mbar_init();
      }
      const uint64_t a0 = sdesc_k_sw32(sa), b0 = sdesc_k_sw32(sb);
      const int tiles = iters / 16;
      for (int t = 0; t < tiles; ++t) {
        const uint32_t d = tmem + (t & 3) * N;
#pragma unroll
        for (int tap = 0; tap < 16; ++tap) {
          const uint64_t ao = (uint64_t)(((tap / 4) * 115 + tap % 4) * 32 >> 4);
          umma_bf16(d, a0 + ao, b0 + (uint64_t)(tap * (N * 32 / 16)), idesc, tap != 0);
        }
        if (variant >= 8) umma_commit(&bars[t & 3]);        // "A stage free"
        if (variant >= 9) umma_commit(&bars[4 + (t & 3)]);  // "accumulator full"
      }
      umma_commit(&bar);
      mbar_wait(&bar, 0);
      long long t1 = clock64();
      if (blockIdx.x == 0) out[0] = t1 - t0;
      iters = 0;
    }
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
  const int smem = 48 * 1024 + N * 512 + 2048 + 32768 + 1024;
  cudaFuncSetAttribute(mma_loop<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 4096;
  static uint8_t* src = nullptr;
  if (!src) cudaMalloc(&src, 4096LL * 16384);
  for (int v = 0; v < 11; ++v) {
    mma_loop<N><<<148, 128, smem>>>(v, iters, d_out, src, 15360);
    mma_loop<N><<<148, 128, smem>>>(v, iters, d_out, src, 15360);
    long long h = 0;
    cudaMemcpy(&h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
    cudaError_t e = cudaGetLastError();
    const double nm = v >= 7 ? (double)(iters / 16 * 16) : v >= 5 ? (double)(iters / 16 * 16 + 1) : v >= 3 ? (double)(iters / 36 * 36 + 1) : (double)iters;
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
