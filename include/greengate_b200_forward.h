/*
 * greengate_b200_forward.h — C ABI of the admitted-batch forward pass
 * (north star subsystem 2) and its building blocks.
 *
 * The reference has no forward pass (its DistilBERT / ResNet-18 exist only as
 * latency/energy constants, pkg/src/greengate/presets.py:50-55; the simulator
 * stands in for the serving backend, servesim.py:137-139, 303-305).  These
 * entry points are what replaces that stand-in.  Same conventions as
 * greengate_b200.h: device pointers owned by the caller, stream-ordered,
 * gg_status return codes.  All tensors are bf16 unless noted; activations are
 * row-major [tokens, features] (DistilBERT) or NHWC (ResNet-18).
 */
#ifndef GREENGATE_B200_FORWARD_H
#define GREENGATE_B200_FORWARD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { GG_ACT_NONE = 0, GG_ACT_RELU = 1, GG_ACT_GELU = 2 };

/* D[M,N] = act(A[M,K] . B[N,K]^T + bias[N] (+ residual[M,N])), bf16 in/out,
 * fp32 accumulation in TMEM (tcgen05.mma, TMA-fed, persistent).  Requires
 * K % 64 == 0, N % 32 == 0, 16-byte aligned rows.  tile_n: 0 = auto, or
 * 64/128/256.  bias is fp32 (may be NULL), residual may be NULL. */
int gg_gemm_bf16(const void* A, int64_t lda, const void* B, int64_t ldb, void* D, int64_t ldd,
                 int64_t M, int64_t N, int64_t K, const float* bias, const void* residual,
                 int64_t ldr, int32_t act, int32_t tile_n, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* GREENGATE_B200_FORWARD_H */
