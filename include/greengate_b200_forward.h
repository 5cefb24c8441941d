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
 *
 * Dynamic batch: every kernel that takes `count_dev` reads the number of
 * valid items (sequences / images) from device memory at launch, so a
 * captured CUDA graph serves whatever the admission step admitted without a
 * host round-trip.  NULL = use the host-side size.
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

/* Output layouts of gg_gemm. */
enum {
  GG_OUT_BF16 = 0,       /* D bf16 [M, ldd] */
  GG_OUT_F32 = 1,        /* D fp32 [M, ldd] (classifier logits for K3) */
  GG_OUT_QKV_HEADS = 2   /* fused-QKV projection: D = bf16 [3][B][H][S][64] planes:
                            Q * 1/sqrt(64), K, and V stored transposed [B][H][64][S] */
};
typedef struct {
  const float* bias;     /* [N] fp32 or NULL */
  const void* residual;  /* bf16 [M, ldr] or NULL, added before the activation */
  int64_t ldr;
  int32_t act;           /* GG_ACT_* */
  int32_t out_mode;      /* GG_OUT_* */
  int32_t seq_len;       /* GG_OUT_QKV_HEADS: S (multiple of 128) */
  int32_t heads;         /* GG_OUT_QKV_HEADS: H, N == 3 * H * 64 */
  int32_t tile_n;        /* 0 = auto, 64 / 128 / 256 */
  int32_t rows_per_item; /* dynamic batch: rows = min(M, *count_dev * rows_per_item) */
  const int32_t* count_dev; /* device item count written by an earlier kernel, or NULL */
} gg_gemm_epilogue;
int gg_gemm(const void* A, int64_t lda, const void* B, int64_t ldb, void* D, int64_t ldd,
            int64_t M, int64_t N, int64_t K, const gg_gemm_epilogue* epilogue, void* stream);

/* LayerNorm folded into the GEMMs around it (no LayerNorm kernel, no
 * normalized activation in HBM).  Row statistics travel as partials: one
 * float2 (mean_i, M2_i) per 128 output columns of a row, plane-major
 * [ln_width / 128][M].
 *   out_stats  this GEMM's output rows (bf16-rounded values): written
 *   a_stats    A holds RAW rows h; the GEMM computes LN(h) W^T + b as
 *              rstd (h W'^T) - rstd mean s_j + c_j, with W' = W diag(gamma)
 *              (the B operand), a_colsum = s_j = sum_k W'_jk and the bias
 *              c_j = b_j + sum_k beta_k W_jk (transformers LayerNorm -> Linear)
 *   r_stats    the residual holds RAW rows h; it is added as
 *              (h - mean) rstd r_gamma + r_beta
 * Only the CTA-pair TMA-epilogue path (N % 256 == 0, M >= 4096) supports it
 * (GG_ERR_UNSUPPORTED otherwise). */
typedef struct {
  const float* a_stats;
  const float* a_colsum;
  const float* r_stats;
  const float* r_gamma;
  const float* r_beta;
  float* out_stats;
  int32_t ln_width;      /* LayerNorm width (768), a multiple of 128 */
  float eps;             /* LayerNorm epsilon */
} gg_gemm_ln_params;
int gg_gemm_ln(const void* A, int64_t lda, const void* B, int64_t ldb, void* D, int64_t ldd,
               int64_t M, int64_t N, int64_t K, const gg_gemm_epilogue* epilogue,
               const gg_gemm_ln_params* ln, void* stream);

/* Tile-level dependencies between consecutive forward kernels, instead of the
 * grid-wide wait of programmatic dependent launch.  Rows are grouped in units
 * of 128 (one DistilBERT sequence); every kernel of the chain counts, per unit,
 * the column tiles (GEMM) or heads (attention) it has finished and published.
 *   wait    the producing kernel's counters [units], or NULL: grid-wide wait on
 *           the stream predecessor (the first kernel of a chain)
 *   need    unit u is ready when wait[u] >= need (the producer's tiles per unit)
 *   signal  this kernel's counters [units] (+1 per finished tile / head), or NULL
 *   go      chain flag: the first kernel sets it to 1 after its grid-wide wait;
 *           the others wait for it before reading count_dev
 *   tiles   this launch's tile counter (GEMM): tiles are claimed dynamically in
 *           row-block order, so CTAs that start early take more; NULL = static
 * The caller zeroes every counter and `go` before the chain (gg_zero_async).
 * Consumers must run after their producers in the same stream; a kernel whose
 * CTAs are all resident only waits on kernels launched before it, so the chain
 * cannot deadlock.  Rows must be consumed in whole units (rows_per_item % 128). */
typedef struct {
  const int32_t* wait;
  int32_t need;
  int32_t* signal;
  int32_t* go;
  int32_t* tiles;
} gg_dep;
int gg_gemm_dep(const void* A, int64_t lda, const void* B, int64_t ldb, void* D, int64_t ldd,
                int64_t M, int64_t N, int64_t K, const gg_gemm_epilogue* epilogue,
                const gg_gemm_ln_params* ln /* or NULL */, const gg_dep* dep, void* stream);
/* DistilBERT's feed-forward block as ONE persistent CTA-pair kernel, with the
 * LayerNorm folding of gg_gemm_ln:
 *   H = gelu(LN1(A) W1^T + b1)     (W1 = W1' = W1 diag(gamma1), colsum1 / bias1
 *                                   the folded column sums / bias, a_stats = A's
 *                                   row statistics partials)
 *   Y = H W2^T + bias2 + LN1(A)     (the residual LayerNorm'd on the fly with
 *                                   r_stats = a_stats, ln_gamma / ln_beta)
 *   out_stats = Y's row statistics partials
 * A [M, d], W1 [F, d], H [M, F] (workspace), W2 [d, F], Y [M, d] bf16; d <= 768
 * and F <= 3072 multiples of 256, M a multiple of 128.  lin2 tiles wait per
 * 128-row unit for that unit's lin1 tiles (ready[M / 128], zeroed by the caller
 * before the launch, like the tile counter tiles[1]); tiles of both GEMMs are
 * claimed from one queue, so the two partial last waves merge. */
int gg_ffn_pair(const void* A, const void* W1, void* H, const void* W2, void* Y, int64_t M, int32_t d,
                int32_t F, const int32_t* count_dev, int32_t rows_per_item, const float* bias1,
                const float* colsum1, const float* a_stats, const float* bias2,
                const float* r_stats, const float* ln_gamma, const float* ln_beta,
                float* out_stats, float eps, int32_t* ready, int32_t* tiles, void* stream);
/* cudaMemsetAsync(ptr, 0, bytes) on the stream (counter reset, graph-capturable). */
int gg_zero_async(void* ptr, int64_t bytes, void* stream);

/* Allocate this device's stream-K workspace (48 MB fp32 partial tiles + 2 MB
 * counters) now, outside any CUDA graph capture.  gg_gemm / gg_conv2d split
 * their (tile, k-block) space evenly over the SMs when the tile count leaves a
 * partly empty last wave; inside a capture without a reserved workspace they
 * run data-parallel.  One stream per device at a time (like the activations). */
int gg_streamk_reserve(void);
/* Stream-K policy: 0 = never (default: on B200 the fixup's partial-tile reads
 * cost more than the last-wave imbalance they remove at the DistilBERT / ResNet
 * shapes), -1 = by the wave model, 1 = whenever the grid has >= 2 k-blocks per
 * SM (tests).  Returns the previous policy. */
int gg_streamk_mode(int32_t mode);

/* Multi-head self-attention for head dim 64 on the GG_OUT_QKV_HEADS planes:
 * ctx[b*S + s, h*64 + d] = softmax(Q K^T + mask) V, one CTA per (b, h), both
 * products on tcgen05 with the scores and the output in TMEM.  mask: int32
 * [B, S] (0 = masked key, DistilBERT's masked_fill with finfo.min) or NULL.
 * Requires S == 128. */
int gg_attention(const void* qkv, const int32_t* mask, void* ctx, int64_t ldc, int32_t batch,
                 int32_t heads, int32_t seq_len, const int32_t* count_dev, void* stream);
/* gg_attention with tile-level dependencies (gg_dep; unit = sequence b: waits
 * for wait[b] >= need before loading (b, h), adds 1 to signal[b] per head). */
int gg_attention_dep(const void* qkv, const int32_t* mask, void* ctx, int64_t ldc, int32_t batch,
                     int32_t heads, int32_t seq_len, const int32_t* count_dev, const gg_dep* dep,
                     void* stream);

/* y = LayerNorm(x) * gamma + beta over rows of width `width` (fp32 statistics),
 * bf16 in/out; eps as in the model config (DistilBERT 1e-12). */
int gg_layernorm(const void* x, int64_t ldx, void* y, int64_t ldy, const float* gamma,
                 const float* beta, int64_t rows, int32_t width, float eps,
                 const int32_t* count_dev, int32_t rows_per_item, void* stream);

/* DistilBERT classification head in one launch (replaces gg_layernorm of the CLS
 * rows + the pre_classifier and classifier GEMMs): for each of `rows` CLS rows
 * (row r at hidden + r * ld_rows, bf16 [768]): x = LayerNorm(row) (skipped when
 * ln_gamma is NULL), pooled = bf16(ReLU(x W_pre^T + b_pre)), logits[r, :labels] =
 * pooled W_cls^T + b_cls (fp32).  W_pre bf16 [768, 768], W_cls bf16 [labels, 768].
 * scratch / arrivals: reserved (may be NULL; the classifier partials are reduced
 * inside a thread-block cluster).  Deterministic. */
int gg_cls_head(const void* hidden, int64_t ld_rows, const float* ln_gamma, const float* ln_beta,
                float eps, const void* w_pre, const float* b_pre, const void* w_cls,
                const float* b_cls, int32_t labels, float* logits, int64_t ld_logits, int32_t rows,
                int32_t max_rows, const int32_t* count_dev, float* scratch, int32_t* arrivals,
                void* stream);
int64_t gg_cls_head_scratch_bytes(int32_t max_rows);

/* Persistent kernels (GEMMs, attention, span convolutions) launched or captured
 * after this call size their grids to (SM count - n) CTAs, n even: the pipelined
 * serving loop keeps a TPC free for the control chain running beside the
 * forward.  Returns the previous value, or -1 for an invalid n. */
int gg_set_sm_reserve(int32_t n);

/* DistilBERT embeddings: y[t] = LayerNorm(word[ids[t]] + pos[t % seq_len]) (bf16 tables). */
int gg_embed_layernorm(const int32_t* ids, const void* word, const void* pos, void* y,
                       const float* gamma, const float* beta, int64_t tokens, int32_t seq_len,
                       int32_t width, float eps, const int32_t* count_dev, void* stream);

/* Gathers the token ids (and attention masks) of a served batch from a
 * resident request pool: ids[i, :] = pool_ids[batch_ids[i] % pool_size, :]. */
int gg_token_gather(const int32_t* pool_ids, const int32_t* pool_mask, int64_t pool_size,
                    const int32_t* batch_ids, const int32_t* count_dev, int32_t B,
                    int32_t seq_len, int32_t* ids, int32_t* mask, void* stream);

/* ---- ResNet-18 (NHWC bf16) ------------------------------------------------ */
/* Implicit-GEMM convolution on tcgen05: y[n,ho,wo,co] = relu?(sum_{r,s,c}
 * x[n, ho*stride-pad+r, wo*stride-pad+s, c] * w[co, (r*S+s)*C + c] + bias[co]
 * (+ residual[n,ho,wo,co])).  w is BN-folded, [Cout, Kpad] with Kpad a
 * multiple of 64 >= R*S*C (zero tail); C % 8 == 0, Cout % 64 == 0. */
int gg_conv2d(const void* x, int32_t N, int32_t H, int32_t W, int32_t C, const void* w,
              int32_t Cout, int32_t R, int32_t S, int32_t stride, int32_t pad, int32_t Kpad,
              const float* bias, const void* residual, int32_t relu, void* y, int32_t pad_hi,
              int32_t out_pad, const int32_t* count_dev, void* stream);
/* out_pad = 1: y (and residual) are zero-bordered [N, Ho+2, Wo+2, Cout]
 * buffers written at (+1, +1) — the layout gg_conv3x3_padded consumes. */
/* 3x3 / stride 1 convolution on zero-padded activations x [N, H+2, W+2, C]
 * writing y [N, H+2, W+2, Cout] (borders written as zeros): all nine taps are
 * shifted views of ONE TMA-loaded span per 64-channel block.  w is BN-folded
 * [Cout, C/64, 3, 3, 64] (K order: channel block, tap, channel); C, Cout % 64
 * == 0; residual (optional) in the same padded layout. */
/* First block of a ResNet stage: conv1 3x3 / stride 2 (+ folded BN, ReLU) on the
 * previous stage's zero-bordered [N, H, W, C] buffer fused with the 1x1 / stride-2
 * downsample (+ folded BN, no ReLU) of the same input — the downsample reads the
 * 3x3's centre-tap tiles.  w: [Cout, 9*C] (r, s, c order), w_ds: [Cout, C]; y and
 * y_ds zero-bordered [N, Ho+2, Wo+2, Cout].  C % 64 == 0, Cout % 128 == 0. */
int gg_conv2d_ds(const void* x, int32_t N, int32_t H, int32_t W, int32_t C, const void* w,
                 int32_t Cout, const float* bias, void* y, const void* w_ds, const float* bias_ds,
                 void* y_ds, int32_t in_shared, int32_t out_shared, const int32_t* count_dev,
                 void* stream);

/* 3x3 / 1 span conv (as gg_conv3x3_padded) on the shared-border layout: per image
 * [H+1, W+1] with one zero row and column (the left / top neighbours of an image's
 * first column / row are the previous row's / image's zeros), after a zero margin of
 * W+2 rows; x, residual and y point at the margin.  ~15-30 % fewer positions than
 * [H+2, W+2] at the 28 / 14 / 7 maps of ResNet layers 2-4. */
int gg_conv3x3_shared(const void* x, int32_t N, int32_t H, int32_t W, int32_t C, const void* w,
                      int32_t Cout, const float* bias, const void* residual, int32_t relu, void* y,
                      const int32_t* count_dev, void* stream);

int gg_conv3x3_padded(const void* x, int32_t N, int32_t H, int32_t W, int32_t C, const void* w,
                      int32_t Cout, const float* bias, const void* residual, int32_t relu,
                      void* y, const int32_t* count_dev, void* stream);
/* (gg_conv2d: pad = top/left padding, pad_hi = bottom/right padding, -1 = same as pad.)
 * A-operand paths: C % 64 == 0 -> one TMA im2col load per (tap, 64 channels);
 * C == 16 -> TMA im2col, 4 taps per 64-wide k-block (the space-to-depth stem);
 * otherwise a cp.async gather. */
/* fp32 NCHW image batch -> bf16 NHWC with channels zero-padded to cpad (% 8). */
int gg_nchw_to_nhwc(const float* x, int32_t N, int32_t C, int32_t H, int32_t W, int32_t cpad,
                    void* y, void* stream);
/* fp32 NCHW RGB batch -> bf16 space-to-depth(2) NHWC, 16 channels
 * (y[n, i, j, (dy*2+dx)*3 + c] = x[n, c, 2i+dy, 2j+dx]; channels 12..15 = 0).
 * ResNet-18's 7x7/2 stem conv equals a 4x4/1 conv (pad 2 / 1) over it.
 * padded = 1: write the interior of a zero-bordered [N, H/2+3, W/2+3, 16]
 * buffer at (+2, +2) — the input layout of gg_stem_s2d_span — PRE-SWIZZLED:
 * cell q (linear index in the padded buffer) has its two 16-byte halves
 * (channels 0-7 / 8-15) swapped when bit 2 of q is set, so that a linear copy
 * into shared memory is the tensor core's SWIZZLE_32B operand layout. */
int gg_nchw_to_s2d16(const float* x, int32_t N, int32_t H, int32_t W, int32_t padded, void* y,
                     void* stream);
/* ResNet-18 stem (conv1 + bn1 + relu) as a span convolution: 4x4 / 1 over the
 * padded space-to-depth input x [N, Hs+3, Ws+3, 16] (Hs = H/2), w BN-folded
 * [64, 4, 4, 16] (gg_nchw_to_s2d16 cell order), y dense [N, Hs, Ws, 64]. */
int gg_stem_s2d_span(const void* x, int32_t N, int32_t Hs, int32_t Ws, const void* w, int32_t Cout,
                     const float* bias, int32_t relu, void* y, const int32_t* count_dev,
                     void* stream);
/* ResNet-18 stem + max pool in one kernel: conv1 + bn1 + relu as gg_stem_s2d_span, then
 * 3x3 / 2 / pad 1 max pool, without writing the stem output.  Hs, Ws even, Ws <= 128;
 * y = pooled [N, Hs/2, Ws/2, 64]: dense (out_pad 0) or the interior of the shared-border
 * layer-1 layout (out_pad 2, as gg_maxpool3x3s2).  Identical values to
 * gg_stem_s2d_span + gg_maxpool3x3s2 (max is order-free, bf16 rounding monotonic).
 * Replaces model.conv1/bn1/relu/maxpool of torchvision resnet18, which the reference
 * runs through torch (kernel K8). */
int gg_stem_pool_span(const void* x, int32_t N, int32_t Hs, int32_t Ws, const void* w, int32_t Cout,
                      const float* bias, void* y, int32_t out_pad, const int32_t* count_dev,
                      void* stream);
/* Served-batch stem input: image i of the batch = uint8 HWC image
 * pool[batch_ids[i] % pool_size], normalized ((x/255 - mean[c]) / std[c]) into
 * the space-to-depth(2) 16-channel layout of gg_nchw_to_s2d16. */
int gg_stem_gather(const uint8_t* pool, int64_t pool_size, const int32_t* batch_ids,
                   const int32_t* count_dev, int32_t B, int32_t H, int32_t W,
                   const float* mean3, const float* std3, int32_t padded, void* y, void* stream);
/* 3x3 / stride 2 / pad 1 max pool (NHWC, C % 8 == 0); out_pad = 1 writes the
 * interior of a zero-bordered [N, Ho+2, Wo+2, C] buffer, out_pad = 2 the interior of
 * a shared-border buffer ([Wo+2 zero rows][N, Ho+1, Wo+1, C], see gg_conv3x3_shared). */
int gg_maxpool3x3s2(const void* x, int32_t N, int32_t H, int32_t W, int32_t C, void* y,
                    int32_t out_pad, const int32_t* count_dev, void* stream);
/* Global average pool NHWC [N, HW, C] -> [N, C], dividing by denom (0 = HW;
 * a zero-bordered input passes its interior pixel count); C % 64 == 0. */
int gg_avgpool(const void* x, int32_t N, int32_t HW, int32_t C, void* y, int32_t denom,
               const int32_t* count_dev, void* stream);
/* ResNet head in fp32: global average pool of the bf16 NHWC map into
 * pooled [N, C] fp32 (no bf16 rounding), then logits [N, ld_logits] fp32 =
 * pooled . w_fc^T + b_fc with fp32 weights [ncls, C] (torchvision's avgpool +
 * fc, fp32 end to end).  Rows past *count_dev are untouched.  C % 128 == 0,
 * C <= 1536. */
int gg_avgpool_fc(const void* x, int32_t N, int32_t HW, int32_t C, int32_t denom,
                  const float* w_fc, const float* b_fc, int32_t ncls, float* pooled,
                  float* logits, int64_t ld_logits, const int32_t* count_dev, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* GREENGATE_B200_FORWARD_H */
