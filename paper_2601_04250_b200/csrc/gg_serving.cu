// gg_serving.cu — device-side glue of the closed serving loop: FIFO pop, served
// outcome records (the exchange slot), the served-batch K3 epilogue and the
// payload gathers that feed the forward with the admitted requests.
#include <cuda_bf16.h>

#include "gg_common.cuh"
#include "gg_kernels.h"
#include "gg_act.cuh"
#include "gg_tc.cuh"

namespace gg {

__device__ __forceinline__ uint64_t now_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// One block: pops n requests and copies the ring slots [head, head+n) out.
// Without a batching window n = min(B, depth).  With one (Path B,
// batch_flush_policy servesim.py:148-162) the batch flushes when it is full
// (n = B) or when the oldest pending request has waited the window in trace
// time (n = depth); otherwise nothing is popped this step.  The trace clock is
// the arrival time of the last decided row (after the trace is exhausted the
// batching timer fires: clock = oldest enqueue + window); it is kept in
// f->clock (monotone) for the served outcomes' latency.
__global__ void fifo_pop_kernel(gg_fifo* f, const int32_t* ring, const uint64_t* ring_ns,
                                int32_t* ids, uint64_t* ns, int32_t* count, int B,
                                const double* now_trace, double window_s) {
  griddep_wait();   // PDL: the predecessor has completed and flushed
  griddep_launch();
  __shared__ int64_t head_s, n_s;
  if (threadIdx.x == 0) {
    const int64_t depth = f->tail - f->head;
    const int64_t mask = f->capacity - 1;
    head_s = f->head;
    int64_t n = depth < B ? depth : B;
    if (now_trace) {
      const int64_t cur = f->cursor < f->trace_len ? f->cursor : f->trace_len;
      double clock = cur > 0 ? now_trace[cur - 1] : 0.0;
      if (window_s > 0.0 && depth > 0 && depth < B) {
        const double oldest = now_trace[ring[head_s & mask]];
        const double deadline = f64_sub(window_s, 1e-12);   // servesim.py:_TIME_EPS
        if (f->cursor >= f->trace_len) {
          const double fire = f64_add(oldest, window_s);       // the batch timer
          clock = fire > clock ? fire : clock;
        } else if (!(f64_sub(clock, oldest) >= deadline)) {
          n = 0;
        }
      }
      f->clock = clock > f->clock ? clock : f->clock;
    }
    n_s = n;
  }
  __syncthreads();
  const int64_t n = n_s, mask = f->capacity - 1;
  for (int i = threadIdx.x; i < B; i += blockDim.x) {
    if (i < n) {
      const int64_t slot = (head_s + i) & mask;
      ids[i] = ring[slot];
      if (ns) ns[i] = ring_ns ? ring_ns[slot] : 0ull;
    } else {
      ids[i] = -1;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    *count = (int32_t)n;
    f->head = head_s + n;
  }
}

// Exchange slot of one rank's step (layout: GG_SLOT_LEN in greengate_b200.h).
__global__ void served_outcomes_kernel(const gg_fifo* f, const int32_t* count, const uint64_t* ns,
                                       gg_outcome_model m, const gg_batch_info* info, double* slot,
                                       int B, const int32_t* ids, const double* now_trace,
                                       double* latency_row) {
  griddep_wait();   // PDL: the predecessor has completed and flushed
  griddep_launch();
  const int n = *count;
  const int64_t depth = f->tail - f->head;            // after the pop
  const double qd = (double)(depth + f->extra_depth);
  const double dn = (double)(n > 0 ? n : 1);
  // servesim.py:303-304: service = base + per_item * n ; joules each = (base_j + per_item_j * n) / n
  const double lat_model = f64_add(m.batch_base_ms, f64_mul(m.per_item_ms, dn));
  const double joules = f64_div(f64_add(m.batch_base_energy_j, f64_mul(m.per_item_energy_j, dn)), dn);
  const uint64_t t = now_ns();
  // GG_LATENCY_TRACE: finish - enqueue in trace time (servesim.py:_maybe_flush /
  // _complete): service_s = (base + per_item * n) / 1000, finish = clock + service_s,
  // latency_ms = (finish - enqueue) * 1000 — the same fp64 operations
  const double finish = f64_add(f->clock, f64_div(lat_model, 1000.0));
  for (int i = threadIdx.x; i < B; i += blockDim.x) {
    double lat = 0.0, jo = 0.0, q = 0.0;
    if (i < n) {
      if (m.measured_latency == GG_LATENCY_TRACE && ids && now_trace)
        lat = f64_mul(f64_sub(finish, now_trace[ids[i]]), 1000.0);
      else if (m.measured_latency == GG_LATENCY_MEASURED && ns)
        lat = (double)(t - ns[i]) * 1e-6;
      else
        lat = lat_model;
      jo = joules;
      q = qd;
      if (latency_row && ids) latency_row[ids[i]] = lat;
    }
    slot[i] = lat;
    slot[B + i] = jo;
    slot[2 * B + i] = q;
  }
  if (threadIdx.x == 0) {
    slot[3 * B] = (double)n;
    slot[3 * B + 1] = (double)depth;
    slot[3 * B + 2] = info ? (double)info->n_decided : 0.0;
    slot[3 * B + 3] = info ? (double)info->n_invalid : 0.0;
    slot[3 * B + 4] = info ? (double)info->n_admitted : 0.0;
    slot[3 * B + 5] = info ? (double)info->n_skipped : 0.0;
    slot[3 * B + 6] = info ? (double)info->snap_queue_depth : 0.0;
    slot[3 * B + 7] = info ? info->snap_p95_ms : 0.0;
  }
}

// K3 over the served batch (see gg_epilogue in gg_controller.cu): one 128-thread
// block per row; each thread keeps its <= 8 logits in registers, so every
// element costs one fp64 exp (max, sum of exp(x - max), then p = e / sum with
// the argmax taken over p, lowest index on ties, as before).
constexpr int kEpiThreads = 128;
constexpr int kEpiPer = 8;   // K <= 1024 in registers

__device__ __forceinline__ void epi_best(double& best, int& bi, double ob, int oi) {
  if (ob > best || (ob == best && oi < bi)) {
    best = ob;
    bi = oi;
  }
}

__global__ void __launch_bounds__(kEpiThreads) epilogue_served_kernel(const float* logits,
                                                                     const int32_t* count, int k,
                                                                     int64_t ld, const int32_t* ids,
                                                                     int32_t* pred, double* conf,
                                                                     double* probs, int32_t* bpred,
                                                                     double* bconf) {
  griddep_wait();   // PDL: the predecessor has completed and flushed
  griddep_launch();
  __shared__ float red_m[kEpiThreads / 32];
  __shared__ double red_s[kEpiThreads / 32];
  __shared__ double red_b[kEpiThreads / 32];
  __shared__ int red_i[kEpiThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int row = blockIdx.x;
  if (row >= *count) return;
  const float* x = logits + (int64_t)row * ld;
  float xv[kEpiPer];
  float m = -INFINITY;
#pragma unroll
  for (int i = 0; i < kEpiPer; ++i) {
    const int j = tid + i * kEpiThreads;
    xv[i] = j < k ? __ldg(x + j) : -INFINITY;
    m = fmaxf(m, xv[i]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) red_m[warp] = m;
  __syncthreads();
#pragma unroll
  for (int w = 0; w < kEpiThreads / 32; ++w) m = fmaxf(m, red_m[w]);
  const double md = (double)m;
  double ev[kEpiPer];
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < kEpiPer; ++i) {
    const int j = tid + i * kEpiThreads;
    ev[i] = j < k ? exp((double)xv[i] - md) : 0.0;
    s += ev[i];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) red_s[warp] = s;
  __syncthreads();
  s = 0.0;
#pragma unroll
  for (int w = 0; w < kEpiThreads / 32; ++w) s += red_s[w];
  const double inv = 1.0 / s;
  double best = -1.0;
  int bi = 0x7fffffff;
#pragma unroll
  for (int i = 0; i < kEpiPer; ++i) {
    const int j = tid + i * kEpiThreads;
    if (j < k) {
      const double pj = ev[i] * inv;
      if (probs) probs[(int64_t)row * k + j] = pj;
      epi_best(best, bi, pj, j);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
    epi_best(best, bi, __shfl_xor_sync(0xffffffffu, best, o), __shfl_xor_sync(0xffffffffu, bi, o));
  if (lane == 0) {
    red_b[warp] = best;
    red_i[warp] = bi;
  }
  __syncthreads();
  if (tid == 0) {
#pragma unroll
    for (int w = 1; w < kEpiThreads / 32; ++w) epi_best(best, bi, red_b[w], red_i[w]);
    const int id = ids[row];
    if (pred) pred[id] = bi;
    if (conf) conf[id] = best;
    if (bpred) bpred[row] = bi;
    if (bconf) bconf[row] = best;
  }
}

// uint8 HWC pool image -> normalized, space-to-depth(2) fp16 NHWC with 16
// channels: y[n, y, x, (dy*2 + dx)*3 + c] = norm(img[2y+dy, 2x+dx, c]), channels
// 12..15 zero.  The ResNet stem (7x7/2 conv) then runs as a 4x4/1 conv over it.
// One thread per output (s2d) pixel: 4 x 3 bytes in, 32 bytes out.
// Destination cell of s2d pixel (yy, xx): dense [N, Ho, Wo, 16], or the
// interior of the zero-bordered [N, Ho+3, Wo+3, 16] buffer (2 before, 1 after)
// that gg_stem_s2d_span reads.
__device__ __forceinline__ int64_t s2d_index(int n, int yy, int xx, int Ho, int Wo, int padded) {
  if (!padded) return ((int64_t)n * Ho + yy) * Wo + xx;
  return ((int64_t)n * (Ho + 3) + yy + 2) * (Wo + 3) + xx + 2;
}

// Store one 32-byte s2d cell.  The padded layout is pre-swizzled for the span
// stem's SWIZZLE_32B operand: cell q keeps its two 16-byte halves swapped when
// bit 2 of q is set (smem address bit 7 of row q within a 256-B atom), so a
// linear bulk copy of any 8-row-aligned span lands as the swizzled tile.
__device__ __forceinline__ void store_s2d_cell(act_t* y, int64_t q, const uint4& lo,
                                               const uint4& hi, int padded) {
  uint4* dst = reinterpret_cast<uint4*>(y + q * 16);
  const bool swap = padded && ((q >> 2) & 1);
  dst[0] = swap ? hi : lo;
  dst[1] = swap ? lo : hi;
}

// One block per (image, kGatherRows s2d rows): the 2 * kGatherRows source image
// rows are staged in shared memory with 16-byte loads (all issued before the
// first use) when aligned, then each thread builds s2d pixels from shared memory
// and writes 32 contiguous bytes (consecutive threads -> consecutive pixels).
constexpr int kGatherThreads = 128;
constexpr int kGatherRows = 4;

__global__ void __launch_bounds__(kGatherThreads) stem_gather_kernel(
    const uint8_t* __restrict__ pool, int64_t pool_size, const int32_t* ids, const int32_t* count,
    int B, int H, int W, float m0, float m1, float m2, float s0, float s1, float s2, int padded,
    act_t* __restrict__ y) {
  extern __shared__ __align__(16) uint8_t rows[];   // [2 * kGatherRows][W * 3]
  // the normalization of a uint8 value is one of 3 x 256 fp16 results: built once
  // per block with the exact arithmetic, then looked up (12 fp32 divisions per
  // cell made this kernel issue-bound).  It depends on nothing the predecessor
  // writes, so it is built before the PDL wait, overlapping the predecessor's tail.
  __shared__ act_t lut[3][256];
  {
    const float mean[3] = {m0, m1, m2}, sd[3] = {s0, s1, s2};
    for (int i = threadIdx.x; i < 3 * 256; i += kGatherThreads) {
      const int c = i >> 8, xv = i & 255;
      lut[c][xv] = float2act(((float)xv * (1.0f / 255.0f) - mean[c]) / sd[c]);
    }
  }
  griddep_wait();   // PDL: the predecessor has completed and flushed
  griddep_launch();
  const int n_valid = count ? min(B, __ldg(count)) : B;
  const int n = blockIdx.y, yy0 = blockIdx.x * kGatherRows;
  if (n >= n_valid) return;
  const int Ho = H / 2, Wo = W / 2;
  const int nrows = min(kGatherRows, Ho - yy0);
  const int64_t img = ids ? (int64_t)__ldg(ids + n) % pool_size : n;
  const int rb = W * 3;
  const uint8_t* src = pool + (img * H + 2 * yy0) * (int64_t)rb;   // 2 * nrows consecutive rows
  const int bytes = 2 * nrows * rb;
  if (((reinterpret_cast<uintptr_t>(src) | (uintptr_t)rb) & 15) == 0) {
    const uint4* s4 = reinterpret_cast<const uint4*>(src);
    for (int i = threadIdx.x; i < bytes / 16; i += kGatherThreads) reinterpret_cast<uint4*>(rows)[i] = __ldg(s4 + i);
  } else {
    for (int i = threadIdx.x; i < bytes; i += kGatherThreads) rows[i] = __ldg(src + i);
  }
  __syncthreads();
  for (int cell = threadIdx.x; cell < nrows * Wo; cell += kGatherThreads) {
    const int r = cell / Wo, xx = cell - r * Wo;
    __align__(16) act_t v[16];
#pragma unroll
    for (int dy = 0; dy < 2; ++dy) {
      const uint8_t* row = rows + (2 * r + dy) * rb + 2 * xx * 3;
#pragma unroll
      for (int i = 0; i < 6; ++i) {  // (dx, c) pairs of this input row
        const int c = i % 3, dx = i / 3;
        v[(dy * 2 + dx) * 3 + c] = lut[c][row[i]];
      }
    }
#pragma unroll
    for (int e = 12; e < 16; ++e) v[e] = float2act(0.0f);
    store_s2d_cell(y, s2d_index(n, yy0 + r, xx, Ho, Wo, padded), reinterpret_cast<uint4*>(v)[0],
                   reinterpret_cast<uint4*>(v)[1], padded);
  }
}

// fp32 NCHW (already normalized) -> the same space-to-depth(2) 16-channel layout.
__global__ void nchw_to_s2d16_kernel(const float* __restrict__ x, int N, int H, int W, int padded,
                                     act_t* __restrict__ y) {
  const int Ho = H / 2, Wo = W / 2;
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= (int64_t)N * Ho * Wo) return;
  const int n = (int)(p / ((int64_t)Ho * Wo));
  const int rem = (int)(p - (int64_t)n * Ho * Wo);
  const int yy = rem / Wo, xx = rem - yy * Wo;
  const int64_t q = s2d_index(n, yy, xx, Ho, Wo, padded);
  __align__(16) act_t v[16];
#pragma unroll
  for (int dy = 0; dy < 2; ++dy)
#pragma unroll
    for (int dx = 0; dx < 2; ++dx)
#pragma unroll
      for (int c = 0; c < 3; ++c)
        v[(dy * 2 + dx) * 3 + c] =
            float2act(__ldg(x + (((int64_t)n * 3 + c) * H + 2 * yy + dy) * W + 2 * xx + dx));
#pragma unroll
  for (int e = 12; e < 16; ++e) v[e] = float2act(0.0f);
  store_s2d_cell(y, q, reinterpret_cast<uint4*>(v)[0], reinterpret_cast<uint4*>(v)[1], padded);
}

__global__ void token_gather_kernel(const int32_t* pool_ids, const int32_t* pool_mask,
                                    int64_t pool_size, const int32_t* ids, const int32_t* count,
                                    int B, int S, int32_t* out_ids, int32_t* out_mask) {
  griddep_wait();   // PDL: the predecessor has completed and flushed
  griddep_launch();
  const int n_valid = count ? min(B, __ldg(count)) : B;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)n_valid * S) return;
  const int n = (int)(t / S), s = (int)(t - (int64_t)n * S);
  const int64_t src = ((int64_t)__ldg(ids + n) % pool_size) * S + s;
  out_ids[t] = pool_ids[src];
  if (out_mask) out_mask[t] = pool_mask ? pool_mask[src] : 1;
}

// ---- open-loop arm (servesim.py:231-240) ----------------------------------
// With the controller disabled the reference admits every arrival and routes
// it statically: ALL_BATCHED -> BATCHED; THRESHOLD_ON_QUEUE -> BATCHED iff the
// queue depth exceeds the threshold, else DIRECT; ALL_DIRECT -> DIRECT.  No
// score is read or validated.  The controller state sees what decide() of an
// always-admitting controller leaves (counters, the snapshot's normalizer
// observes), exactly like the other ranks' slots are applied by K2, so
// multi-GPU replicas stay identical; the ledger is fed by K2 as
// servesim.py:272-273 feeds it.
__global__ void admit_open_kernel(gg_params p, gg_state* st, gg_fifo* f, int32_t* ring,
                                  uint64_t* ring_ns, int64_t window, uint8_t* decision,
                                  gg_batch_info* info) {
  griddep_wait();
  griddep_launch();
  __shared__ int64_t row0_s, n_s, tail_s, depth_s;
  __shared__ uint8_t code_s;
  if (threadIdx.x == 0) {
    const int64_t row0 = f->cursor;
    const int64_t left = f->trace_len - row0;
    const int64_t n = left < window ? (left > 0 ? left : 0) : window;
    const int64_t depth = f->tail - f->head;
    const int64_t qd = depth + f->extra_depth;
    uint8_t code = GG_DECISION_DIRECT;
    if (p.routing == GG_ROUTE_ALL_BATCHED) code = GG_DECISION_BATCHED;
    else if (p.routing == GG_ROUTE_THRESHOLD_ON_QUEUE && qd > (int64_t)p.queue_threshold)
      code = GG_DECISION_BATCHED;
    row0_s = row0; n_s = n; tail_s = f->tail; depth_s = depth; code_s = code;
    double e = 0.0, c = 0.0;
    const double p95 = st->p95_current;
    const double fill0 = f64_div((double)depth, (double)f->batch_cap);
    const double fill = fill0 < 1.0 ? fill0 : 1.0;
    if (n > 0) {   // decide()'s normalize() observes (controller.py:316-325) + counters
      gg_channel ce = st->n_energy, cq = st->n_queue_depth, cp = st->n_p95_ms;
      e = st->samples_seen > 0 ? ch_normalize(ce, st->ewma_joules_per_request) : 0.0;
      const double qn = ch_normalize(cq, (double)qd), pn = ch_normalize(cp, p95);
      c = f64_div(f64_add(f64_add(qn, pn), fill), 3.0);
      st->n_energy = ce; st->n_queue_depth = cq; st->n_p95_ms = cp;
      st->admitted_total += n;
    }
    if (info) {
      info->n_admitted = n; info->n_skipped = 0; info->n_invalid = 0; info->first_invalid = -1;
      info->energy = e; info->congestion = c; info->n_decided = n;
      info->snap_queue_depth = qd; info->snap_p95_ms = p95; info->snap_batch_fill = fill;
    }
  }
  __syncthreads();
  const int64_t n = n_s, row0 = row0_s, tail = tail_s, depth = depth_s;
  const int64_t cap = f->capacity, mask = cap - 1;
  const uint8_t code = code_s;
  const uint64_t t = now_ns();
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    decision[row0 + i] = code;
    if (depth + i < cap) {
      const int64_t slot = (tail + i) & mask;
      ring[slot] = (int32_t)(row0 + i);
      if (ring_ns) ring_ns[slot] = t;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int64_t room = cap - depth;
    const int64_t stored = n < room ? n : room;
    f->tail = tail + stored;
    if (n > stored) f->overflow += n - stored;
    f->cursor = row0 + n;
  }
}

// ---- fallback answers (servesim.py:246-256) ---------------------------------
// Every decided row gets the reference's answer: top_class() of its scores
// (first max, workload.py:42-43).  Accounting as in Simulation._complete:
// admitted rows are correct iff top == label; a skipped row is correct iff
// top == label AND its fallback coin >= fallback_degradation, where the coins
// are the `_fb_rng` stream (drawn on the host, never on the device) consumed in
// trace order by exactly the skipped rows with top == label (the `and`
// short-circuits).  One 8-CTA cluster: the top classes of up to kFbSuper rows
// at a time are computed by all 64 warps (a thread per row for K <= 32, else a
// warp per row) and stored into CTA 0's shared memory over DSMEM; after a
// cluster barrier CTA 0 scans the coin flags in trace order, 256 rows per
// block scan.  (As one block the K = 1000 ResNet window -- 112 rows x 8 KB --
// took ~42 us of a 430 us serving step on a single SM's load bandwidth.)
constexpr int kFbThreads = 256;
constexpr int kFbCluster = 8;
constexpr int kFbSuper = 4096;

__global__ void __cluster_dims__(kFbCluster, 1, 1) __launch_bounds__(kFbThreads) fallback_kernel(
    const double* __restrict__ scores, int k, int64_t stride, const int32_t* __restrict__ labels,
    const uint8_t* __restrict__ decision, const gg_fifo* f, const gg_batch_info* info,
    int64_t row0_arg, int64_t n_arg, const double* __restrict__ coins, int64_t* coin_cursor,
    double degradation, int32_t* answer, uint8_t* correct) {
  griddep_wait();
  griddep_launch();
  __shared__ int32_t top_s[kFbSuper];         // CTA 0's copy is the one written
  __shared__ int32_t warp_tot[kFbThreads / 32];
  __shared__ int64_t base_s;
  const uint32_t crank = tc::cluster_ctarank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gthread = (int)crank * kFbThreads + tid;
  const int gwarp = gthread >> 5;
  constexpr int kThreadsAll = kFbCluster * kFbThreads, kWarpsAll = kThreadsAll / 32;
  const uint32_t top0 = tc::mapa_shared(tc::smem_u32(top_s), 0);
  int64_t row0 = row0_arg, n = n_arg;
  if (f && info) {            // the window the admission kernel just decided
    n = info->n_decided;
    row0 = f->cursor - n;
  }
  if (crank == 0 && tid == 0) base_s = *coin_cursor;
  for (int64_t s0 = 0; s0 < n; s0 += kFbSuper) {   // uniform across the cluster
    const int sn = (int)min((int64_t)kFbSuper, n - s0);
    if (k <= 32) {
      for (int i = gthread; i < sn; i += kThreadsAll) {
        const double* x = scores + (row0 + s0 + i) * stride;
        double best = x[0];
        int bi = 0;
        for (int j = 1; j < k; ++j) {
          const double v = x[j];
          if (v > best) { best = v; bi = j; }
        }
        tc::st_shared_cluster_s32(top0 + 4u * (uint32_t)i, bi);
      }
    } else {
      for (int i = gwarp; i < sn; i += kWarpsAll) {
        const double* x = scores + (row0 + s0 + i) * stride;
        double best = -INFINITY;
        int bi = 0x7fffffff;
        for (int j0 = lane; j0 < k; j0 += 8 * 32) {   // 8 loads in flight per lane
          double v[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) v[e] = j0 + 32 * e < k ? __ldg(x + j0 + 32 * e) : -INFINITY;
#pragma unroll
          for (int e = 0; e < 8; ++e)   // lanes see ascending j: first max per lane
            if (v[e] > best) { best = v[e]; bi = j0 + 32 * e; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double ob = __shfl_xor_sync(0xffffffffu, best, o);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
          if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
        }
        if (lane == 0) tc::st_shared_cluster_s32(top0 + 4u * (uint32_t)i, bi);
      }
    }
    tc::cluster_sync_all();   // every top of the super-chunk is in CTA 0
    if (crank == 0) {
      for (int c0 = 0; c0 < sn; c0 += kFbThreads) {
        const int cn = min(kFbThreads, sn - c0);
        int flag = 0, top = -1, lab = -1;
        uint8_t dec = GG_DECISION_INVALID;
        const int64_t row = row0 + s0 + c0 + tid;
        if (tid < cn) {
          dec = decision[row];
          top = top_s[c0 + tid];
          lab = labels ? labels[row] : -1;
          flag = (dec == GG_DECISION_SKIP) && (top == lab);
        }
        const unsigned bal = __ballot_sync(0xffffffffu, flag);
        if (lane == 0) warp_tot[warp] = __popc(bal);
        __syncthreads();
        int pre = __popc(bal & ((1u << lane) - 1u)), tot = 0;
#pragma unroll
        for (int w = 0; w < kFbThreads / 32; ++w) {
          if (w < warp) pre += warp_tot[w];
          tot += warp_tot[w];
        }
        if (tid < cn && dec != GG_DECISION_INVALID) {
          if (answer) answer[row] = top;
          if (correct) {
            bool ok = (top == lab);
            if (dec == GG_DECISION_SKIP) ok = flag && coins[base_s + pre] >= degradation;
            correct[row] = ok ? 1 : 0;
          }
        }
        __syncthreads();
        if (tid == 0) base_s += tot;
        __syncthreads();
      }
    }
    tc::cluster_sync_all();   // CTA 0 has read the tops before the next super-chunk
  }
  if (crank == 0 && tid == 0) *coin_cursor = base_s;
}

}  // namespace gg

using namespace gg;


// ---- step record into host-mapped memory (gg_publish_step) -------------------
static __host__ __device__ inline size_t step_rec_conf_off(int B) {
  return (sizeof(gg_step_record) + 4 * (size_t)B + 7) & ~(size_t)7;
}
static __host__ __device__ inline size_t step_rec_bytes(int B, int W) {
  return (step_rec_conf_off(B) + 8 * (size_t)B + (size_t)W + 63) & ~(size_t)63;
}

__global__ void publish_step_kernel(const int32_t* count, const int32_t* pred, const double* conf,
                                    const uint8_t* decision, const gg_batch_info* info,
                                    const gg_fifo* fifo, int B, int W, uint8_t* host, int64_t* seq) {
  griddep_wait();   // PDL: the predecessor has completed and flushed
  griddep_launch();
  const int64_t s = *seq;
  uint8_t* rec = host + (s & 1) * step_rec_bytes(B, W);
  const int n = *count;
  const int64_t nd = info ? info->n_decided : 0;
  const int64_t w0 = fifo->cursor - nd;
  int32_t* rp = reinterpret_cast<int32_t*>(rec + sizeof(gg_step_record));
  double* rc = reinterpret_cast<double*>(rec + step_rec_conf_off(B));
  uint8_t* rd = rec + step_rec_conf_off(B) + 8 * (size_t)B;
  for (int i = threadIdx.x; i < B; i += blockDim.x) {
    rp[i] = i < n ? pred[i] : -1;
    rc[i] = i < n ? conf[i] : 0.0;
  }
  for (int i = threadIdx.x; i < W; i += blockDim.x) rd[i] = i < nd ? decision[w0 + i] : (uint8_t)254;
  if (threadIdx.x == 0) {
    gg_step_record h;
    h.count = n;
    h.n_decided = (int32_t)nd;
    h.window_start = w0;
    h.step = s;
    h.reserved = 0;
    *reinterpret_cast<gg_step_record*>(rec) = h;
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) *seq = s + 1;
}

extern "C" {

int gg_fifo_pop(gg_fifo* fifo_dev, const int32_t* ring_ids_dev, const uint64_t* ring_ns_dev,
                int32_t* batch_ids_dev, uint64_t* batch_ns_dev, int32_t* count_dev, int32_t B,
                void* stream) {
  return gg_fifo_pop_windowed(fifo_dev, ring_ids_dev, ring_ns_dev, nullptr, 0.0, batch_ids_dev,
                              batch_ns_dev, count_dev, B, stream);
}

int gg_fifo_pop_windowed(gg_fifo* fifo_dev, const int32_t* ring_ids_dev,
                         const uint64_t* ring_ns_dev, const double* now_dev,
                         double batching_window_s, int32_t* batch_ids_dev,
                         uint64_t* batch_ns_dev, int32_t* count_dev, int32_t B, void* stream) {
  if (!fifo_dev || !ring_ids_dev || !batch_ids_dev || !count_dev || B < 1) return GG_ERR_INVALID_ARGUMENT;
  if (!(batching_window_s >= 0.0) || (batching_window_s > 0.0 && !now_dev)) return GG_ERR_INVALID_ARGUMENT;
  GG_PDL_LAUNCH((fifo_pop_kernel), 1, 256, 0, gg_stream(stream), fifo_dev, ring_ids_dev, ring_ns_dev,
                batch_ids_dev, batch_ns_dev, count_dev, B, now_dev, batching_window_s);
  GG_LAUNCH_OK();
  return GG_OK;
}

int gg_admit_open_stream(const gg_params* params, gg_state* state_dev, gg_fifo* fifo_dev,
                         int32_t* ring_ids_dev, uint64_t* ring_ns_dev, int64_t window,
                         uint8_t* decision_dev, gg_batch_info* info_dev, void* stream) {
  int rc = gg_validate_params(params);
  if (rc != GG_OK) return rc;
  if (!state_dev || !fifo_dev || !ring_ids_dev || !decision_dev || window < 1)
    return GG_ERR_INVALID_ARGUMENT;
  GG_PDL_LAUNCH((admit_open_kernel), 1, 256, 0, gg_stream(stream), *params, state_dev, fifo_dev,
                ring_ids_dev, ring_ns_dev, window, decision_dev, info_dev);
  GG_LAUNCH_OK();
  return GG_OK;
}

int gg_fallback_answers(const double* probs_dev, int32_t k, int64_t row_stride,
                        const int32_t* labels_dev, const uint8_t* decision_dev,
                        const gg_fifo* fifo_dev, const gg_batch_info* info_dev, int64_t row0,
                        int64_t n, const double* coins_dev, int64_t* coin_cursor_dev,
                        double fallback_degradation, int32_t* answer_dev, uint8_t* correct_dev,
                        void* stream) {
  if (!probs_dev || !decision_dev || !coin_cursor_dev || k < 1 || row_stride < k)
    return GG_ERR_INVALID_ARGUMENT;
  if ((fifo_dev == nullptr) != (info_dev == nullptr)) return GG_ERR_INVALID_ARGUMENT;
  if (!fifo_dev && (row0 < 0 || n < 0)) return GG_ERR_INVALID_ARGUMENT;
  if (correct_dev && (!coins_dev || !labels_dev)) return GG_ERR_INVALID_ARGUMENT;
  if (!(fallback_degradation >= 0.0 && fallback_degradation <= 1.0)) return GG_ERR_INVALID_ARGUMENT;
  GG_PDL_LAUNCH((fallback_kernel), kFbCluster, kFbThreads, 0, gg_stream(stream), probs_dev, k, row_stride,
                labels_dev, decision_dev, fifo_dev, info_dev, row0, n, coins_dev, coin_cursor_dev,
                fallback_degradation, answer_dev, correct_dev);
  GG_LAUNCH_OK();
  return GG_OK;
}

int gg_served_outcomes(const gg_fifo* fifo_dev, const int32_t* count_dev,
                       const uint64_t* batch_ns_dev, const gg_outcome_model* model,
                       const gg_batch_info* info_dev, double* slot_dev, int32_t B, void* stream) {
  return gg_served_outcomes_trace(fifo_dev, count_dev, batch_ns_dev, nullptr, nullptr, model,
                                  info_dev, slot_dev, B, nullptr, stream);
}


size_t gg_step_record_bytes(int32_t B, int32_t W) {
  return (B < 1 || W < 1) ? 0 : step_rec_bytes(B, W);
}

int gg_publish_step(const int32_t* count_dev, const int32_t* batch_pred_dev,
                    const double* batch_conf_dev, const uint8_t* decision_dev,
                    const gg_batch_info* info_dev, const gg_fifo* fifo_dev, int32_t B, int32_t W,
                    void* host_records, int64_t* seq_dev, void* stream) {
  if (!count_dev || !batch_pred_dev || !batch_conf_dev || !decision_dev || !info_dev || !fifo_dev ||
      !host_records || !seq_dev || B < 1 || W < 1)
    return GG_ERR_INVALID_ARGUMENT;
  GG_PDL_LAUNCH((publish_step_kernel), 1, 256, 0, gg_stream(stream), count_dev, batch_pred_dev,
                batch_conf_dev, decision_dev, info_dev, fifo_dev, B, W,
                reinterpret_cast<uint8_t*>(host_records), seq_dev);
  GG_LAUNCH_OK();
  return GG_OK;
}

int gg_served_outcomes_trace(const gg_fifo* fifo_dev, const int32_t* count_dev,
                             const uint64_t* batch_ns_dev, const int32_t* batch_ids_dev,
                             const double* now_dev, const gg_outcome_model* model,
                             const gg_batch_info* info_dev, double* slot_dev, int32_t B,
                             double* latency_row_dev, void* stream) {
  if (!fifo_dev || !count_dev || !model || !slot_dev || B < 1) return GG_ERR_INVALID_ARGUMENT;
  if ((model->measured_latency == GG_LATENCY_TRACE && !now_dev) ||
      ((model->measured_latency == GG_LATENCY_TRACE || latency_row_dev) && !batch_ids_dev))
    return GG_ERR_INVALID_ARGUMENT;
  if (model->batch_base_ms < 0 || model->per_item_ms < 0 || model->batch_base_energy_j < 0 ||
      model->per_item_energy_j < 0)
    return GG_ERR_NEGATIVE_MEASUREMENT;
  GG_PDL_LAUNCH((served_outcomes_kernel), 1, 256, 0, gg_stream(stream), fifo_dev, count_dev, batch_ns_dev,
                *model, info_dev, slot_dev, B, batch_ids_dev, now_dev, latency_row_dev);
  GG_LAUNCH_OK();
  return GG_OK;
}

int gg_epilogue_served(const float* logits_dev, const int32_t* count_dev, int32_t B, int32_t k,
                       int64_t ld, const int32_t* batch_ids_dev, int32_t* predicted_dev,
                       double* confidence_dev, double* probs_dev, int32_t* batch_predicted_dev,
                       double* batch_confidence_dev, void* stream) {
  if (!logits_dev || !count_dev || !batch_ids_dev || B < 1 || k < 1 || ld < k)
    return GG_ERR_INVALID_ARGUMENT;
  if (k > kEpiThreads * kEpiPer) return GG_ERR_UNSUPPORTED;
  GG_PDL_LAUNCH((epilogue_served_kernel), B, kEpiThreads, 0, gg_stream(stream), 
      logits_dev, count_dev, k, ld, batch_ids_dev, predicted_dev, confidence_dev, probs_dev,
      batch_predicted_dev, batch_confidence_dev);
  GG_LAUNCH_OK();
  return GG_OK;
}

int gg_stem_gather(const uint8_t* pool, int64_t pool_size, const int32_t* batch_ids,
                   const int32_t* count_dev, int32_t B, int32_t H, int32_t W, const float* mean3,
                   const float* std3, int32_t padded, void* y, void* stream) {
  if (!pool || pool_size < 1 || !mean3 || !std3 || !y || B < 1 || H % 2 || W % 2)
    return GG_ERR_INVALID_ARGUMENT;
  if (2 * kGatherRows * W * 3 > 48 * 1024 || B > 65535) return GG_ERR_UNSUPPORTED;
  GG_PDL_LAUNCH((stem_gather_kernel), dim3((unsigned)((H / 2 + kGatherRows - 1) / kGatherRows), (unsigned)B),
                kGatherThreads, 2 * kGatherRows * W * 3, gg_stream(stream),
      pool, pool_size, batch_ids, count_dev, B, H, W, mean3[0], mean3[1], mean3[2], std3[0],
      std3[1], std3[2], padded, reinterpret_cast<act_t*>(y));
  GG_LAUNCH_OK();
  return GG_OK;
}

int gg_nchw_to_s2d16(const float* x, int32_t N, int32_t H, int32_t W, int32_t padded, void* y,
                     void* stream) {
  if (!x || !y || N < 1 || H % 2 || W % 2) return GG_ERR_INVALID_ARGUMENT;
  const int64_t pixels = (int64_t)N * (H / 2) * (W / 2);
  nchw_to_s2d16_kernel<<<(unsigned)((pixels + 255) / 256), 256, 0, gg_stream(stream)>>>(
      x, N, H, W, padded, reinterpret_cast<act_t*>(y));
  GG_LAUNCH_OK();
  return GG_OK;
}

int gg_token_gather(const int32_t* pool_ids, const int32_t* pool_mask, int64_t pool_size,
                    const int32_t* batch_ids, const int32_t* count_dev, int32_t B,
                    int32_t seq_len, int32_t* ids, int32_t* mask, void* stream) {
  if (!pool_ids || pool_size < 1 || !batch_ids || !ids || B < 1 || seq_len < 1)
    return GG_ERR_INVALID_ARGUMENT;
  const int64_t tokens = (int64_t)B * seq_len;
  GG_PDL_LAUNCH((token_gather_kernel), (unsigned)((tokens + 255) / 256), 256, 0, gg_stream(stream), 
      pool_ids, pool_mask, pool_size, batch_ids, count_dev, B, seq_len, ids, mask);
  GG_LAUNCH_OK();
  return GG_OK;
}

}  // extern "C"
