// tma_bench.cu — per-SM TMA ingress: one CTA per SM streams 2-D boxes of a
// bf16 matrix into a shared-memory ring (no consumer work) and reports bytes
// per SM cycle, for several box shapes / ring depths / source sizes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/_tma_bench tools/tma_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include "../paper_2601_04250_b200/csrc/gg_tc.cuh"

using namespace gg::tc;

__global__ void __launch_bounds__(32, 1) tma_stream(const __grid_constant__ CUtensorMap map, int box_rows,
                                                    int stages, int iters, int total_rows,
                                                    long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[16];
  const int stage_bytes = box_rows * 128;
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) mbar_init(&full[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int nblk = total_rows / box_rows;
    long long t0 = clock64();
    for (int i = 0; i < iters + stages; ++i) {
      const int s = i % stages;
      if (i >= stages) mbar_wait(&full[s], ((i - stages) / stages) & 1);
      if (i < iters) {
        mbar_expect_tx(&full[s], stage_bytes);
        const int blk = (blockIdx.x * 7919 + i * 131) % nblk;
        tma_load_2d(smem + s * stage_bytes, &map, &full[s], 0, blk * box_rows);
      }
    }
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
}

// Same stream with 1-D bulk copies (cp.async.bulk) of contiguous row ranges.
__global__ void __launch_bounds__(32, 1) bulk_stream(const uint8_t* src, int box_rows, int stages,
                                                     int iters, int total_rows, long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[16];
  const int stage_bytes = box_rows * 128;
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) mbar_init(&full[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int nblk = total_rows / box_rows;
    long long t0 = clock64();
    for (int i = 0; i < iters + stages; ++i) {
      const int s = i % stages;
      if (i >= stages) mbar_wait(&full[s], ((i - stages) / stages) & 1);
      if (i < iters) {
        mbar_expect_tx(&full[s], stage_bytes);
        const int blk = (blockIdx.x * 7919 + i * 131) % nblk;
        bulk_load(smem + s * stage_bytes, src + (size_t)blk * stage_bytes, stage_bytes, &full[s]);
      }
    }
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 enc;

int main() {
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  long long* d_out;
  cudaMalloc(&d_out, 148 * sizeof(long long));
  const int sms = 148;
  cudaFuncSetAttribute(tma_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  for (long long mb : {16LL, 1024LL}) {   // L2-resident vs HBM-sized source
    const long long rows = mb * 1024 * 1024 / 128;
    void* src;
    cudaMalloc(&src, rows * 128);
    cudaMemset(src, 0, rows * 128);
    for (int box_rows : {64, 128, 256}) {
      for (int stages : {2, 4, 6}) {
        if (stages * box_rows * 128 > 200 * 1024) continue;
        CUtensorMap map;
        cuuint64_t dims[2] = {64, (cuuint64_t)rows};
        cuuint64_t strides[1] = {128};
        cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
        cuuint32_t estr[2] = {1, 1};
        CUresult er = enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (er != CUDA_SUCCESS) { printf("encode failed %d\n", (int)er); continue; }
        const int iters = 400;
        const int smem = stages * box_rows * 128 + 1024;
        tma_stream<<<sms, 32, smem>>>(map, box_rows, stages, iters, (int)rows, d_out);
        cudaError_t e1 = cudaDeviceSynchronize();
        tma_stream<<<sms, 32, smem>>>(map, box_rows, stages, iters, (int)rows, d_out);
        cudaError_t e2 = cudaDeviceSynchronize();
        if (e1 != cudaSuccess || e2 != cudaSuccess) {
          printf("launch failed: %s / %s\n", cudaGetErrorString(e1), cudaGetErrorString(e2));
          return 1;
        }
        long long h[148];
        cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
        double avg = 0;
        for (int i = 0; i < sms; ++i) avg += h[i];
        avg /= sms;
        const double bpc = (double)iters * box_rows * 128 / avg;
        printf("src %5lld MB  box %3d rows x 128 B  stages %d: %6.1f B/cycle/SM  (%.2f TB/s @1.9GHz)\n",
               mb, box_rows, stages, bpc, bpc * 148 * 1.9e9 / 1e12);
      }
    }
    cudaFuncSetAttribute(bulk_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    for (int box_rows : {64, 128, 256}) {
      for (int stages : {2, 4, 6}) {
        if (stages * box_rows * 128 > 200 * 1024) continue;
        const int iters = 400;
        const int smem = stages * box_rows * 128 + 1024;
        for (int rep = 0; rep < 2; ++rep)
          bulk_stream<<<sms, 32, smem>>>((const uint8_t*)src, box_rows, stages, iters, (int)rows, d_out);
        if (cudaDeviceSynchronize() != cudaSuccess) { printf("bulk launch failed\n"); return 1; }
        long long h[148];
        cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
        double avg = 0;
        for (int i = 0; i < sms; ++i) avg += h[i];
        avg /= sms;
        const double bpc = (double)iters * box_rows * 128 / avg;
        printf("BULK src %5lld MB  %3d rows x 128 B  stages %d: %6.1f B/cycle/SM  (%.2f TB/s @1.9GHz)\n",
               mb, box_rows, stages, bpc, bpc * 148 * 1.9e9 / 1e12);
      }
    }
    cudaFree(src);
  }
  return 0;
}
