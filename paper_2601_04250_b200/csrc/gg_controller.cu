// gg_controller.cu — admission (K1), outcome feedback (K2) and logit epilogue
// (K3) kernels of the gated-inference hot path, plus their C-ABI entry points
// (include/greengate_b200.h).
//
// Compiled with -fmad=false; every controller operation additionally goes
// through the __d*_rn intrinsics in gg_common.cuh, so each fp64 binary op
// rounds exactly like CPython's float op in the reference
// (pkg/src/greengate/controller.py, energy.py, telemetry.py).
#include <math.h>
#include <mutex>
#include <unordered_map>
#include <utility>
#include <stdio.h>
#include <stdlib.h>

#include "gg_common.cuh"
#include "gg_kernels.h"

namespace gg {

// ---------------------------------------------------------------------------
// Workspace layout (zero-filled once; every gg_admit launch leaves it zeroed).
struct AdmitWorkspace {
  unsigned long long vblock_counter;  // reserved (tiles are scanned in blockIdx order)
  unsigned long long done_counter;    // completion ticket; the last block finalizes
  unsigned long long n_skipped;
  unsigned long long n_invalid;
  unsigned long long first_invalid_enc;  // max over (n - row); 0 == none
  unsigned long long reserved[3];
  unsigned long long consts[24];      // split path: BatchConst + FastBlock of this launch
  unsigned long long status[1];       // [num_blocks] decoupled look-back words
};
constexpr size_t kWsHeader = offsetof(AdmitWorkspace, status);
constexpr unsigned long long kFlagAgg = 1ull << 62;
constexpr unsigned long long kFlagPrefix = 2ull << 62;
constexpr unsigned long long kValMask = (1ull << 62) - 1;

__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// A status value packs two 31-bit counters, summed component-wise by plain
// addition (launches are limited to < 2^31 rows): admitted rows in bits 0..30,
// skipped rows in bits 31..61.  Carrying the skip count through the scan
// replaces a per-warp atomic on one global counter (which serialised in L2 at
// 2^26 rows); n_invalid = rows - admitted - skipped.
constexpr unsigned long long kCnt31 = (1ull << 31) - 1;
__device__ __forceinline__ unsigned long long pack_counts(unsigned long long adm, unsigned long long skip) {
  return adm | (skip << 31);
}

// Warp-cooperative decoupled look-back (Merrill & Garland), called by all 32
// lanes of one warp: each round inspects the 32 preceding status words at once,
// stops at the nearest inclusive prefix.  Returns the exclusive prefix.
__device__ unsigned long long lookback_warp(unsigned long long* status, int vb, unsigned long long agg) {
  const int lane = threadIdx.x & 31;
  if (vb == 0) {
    if (lane == 0) st_relaxed(&status[0], kFlagPrefix | agg);
    return 0ull;
  }
  if (lane == 0) st_relaxed(&status[vb], kFlagAgg | agg);
  unsigned long long prefix = 0;
  int base = vb - 1;
  while (true) {
    const int p = base - lane;
    unsigned long long w = kFlagPrefix;   // before block 0: an empty prefix
    if (p >= 0) {
      do {
        w = ld_relaxed(&status[p]);
      } while ((w >> 62) == 0ull);
    }
    const unsigned pm = __ballot_sync(0xffffffffu, (w >> 62) == 2ull);
    const int stop = pm ? __ffs(pm) - 1 : 31;
    unsigned long long v = lane <= stop ? (w & kValMask) : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    prefix += v;
    if (pm) break;
    base -= 32;
  }
  if (lane == 0) st_relaxed(&status[vb], kFlagPrefix | (prefix + agg));
  return prefix;
}

struct AdmitArgs {
  gg_params p;
  gg_state* state;
  const double* probs;
  int64_t n;
  int32_t k;
  int64_t stride;
  const double* now;
  const gg_snapshot* snap;
  uint8_t* decision;
  double* breakdown;
  int32_t* admitted_idx;
  gg_batch_info* info;
  AdmitWorkspace* ws;
  double ln_k;  // math.log(len(xs)) computed on the host with libm (controller.py:142)
  // stream mode (serving loop): rows [fifo->cursor, +n) of a resident trace,
  // admitted trace rows appended to the device FIFO ring.
  gg_fifo* fifo;
  int32_t* ring;
  uint64_t* ring_ns;
  // split path (large batches): per-decide-block packed counts and per-super-
  // block sums (2^super_shift decide blocks each), inside the workspace after
  // the look-back words; zero between launches like the look-back words.
  unsigned long long* split_cnt;
  unsigned long long* super_cnt;
  int super_shift;
};

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Resolve the rows this launch decides: n rows starting at row0.  In stream
// mode the window starts at the FIFO's trace cursor (read before any block
// finishes; the last block advances it).
__device__ __forceinline__ void admit_window(const AdmitArgs& a, int64_t& row0, int64_t& n) {
  if (a.fifo) {
    row0 = a.fifo->cursor;
    const int64_t left = a.fifo->trace_len - row0;
    n = left < a.n ? (left > 0 ? left : 0) : a.n;
  } else {
    row0 = 0;
    n = a.n;
  }
}

// Batch-constant part of decide() (controller.py:316-325).  Within one frozen
// snapshot every valid request sees the same E and C: the first valid
// request's normalize() observes the raw values, later ones re-observe the
// same values (idempotent), so evaluating normalize on a copy of the channels
// yields exactly the per-request values.
struct BatchConst {
  double e, c, p95, fill, t_origin, ewma;
  int64_t qd;
  int64_t samples_seen;
};

__device__ BatchConst batch_constants(const gg_state* st, const gg_snapshot* snap,
                                      const gg_fifo* fifo) {
  BatchConst b;
  b.samples_seen = st->samples_seen;
  b.ewma = st->ewma_joules_per_request;
  b.t_origin = st->t_origin;
  if (snap) {
    b.qd = snap->queue_depth;
    b.p95 = snap->p95_latency_ms;
    b.fill = snap->batch_fill;
  } else if (fifo) {  // serving loop: the FIFO is the queue (servesim.py:208-220 semantics)
    const int64_t depth = fifo->tail - fifo->head;
    b.qd = depth + fifo->extra_depth;
    b.p95 = st->p95_current;
    const double f = f64_div((double)depth, (double)fifo->batch_cap);
    b.fill = f < 1.0 ? f : 1.0;
  } else {  // default congestion source (controller.py:295-300; gateway.py:58-64)
    b.qd = st->queue_depth;
    b.p95 = st->p95_current;
    b.fill = 0.0;
  }
  gg_channel ce = st->n_energy, cq = st->n_queue_depth, cp = st->n_p95_ms;
  b.e = (b.samples_seen > 0) ? ch_normalize(ce, b.ewma) : 0.0;
  double qn = ch_normalize(cq, (double)b.qd);
  double pn = ch_normalize(cp, b.p95);
  b.c = f64_div(f64_add(f64_add(qn, pn), b.fill), 3.0);
  return b;
}

// _validate_distribution + utility proxy, one streaming pass over the row in
// index order (controller.py:126-148).
struct RowAcc {
  bool ok = true;
  bool first = true;
  NeumaierSum tot, h;
  double mx = 0.0;
  __device__ __forceinline__ void add(double x, bool entropy) {
    if (!isfinite(x) || x < 0.0) ok = false;
    tot.add(x);
    if (entropy) {
      if (x > 0.0) h.add(f64_mul(x, log(x)));
    } else {
      if (first || x > mx) mx = x;
      first = false;
    }
  }
  __device__ __forceinline__ bool finish(int k, bool entropy, double ln_k, double& u) const {
    if (!ok || k < 2) return false;
    if (fabs(f64_sub(tot.result(), 1.0)) > 1e-9) return false;
    if (entropy) u = clamp01(f64_div(-h.result(), ln_k));
    else u = f64_sub(1.0, mx);
    return true;
  }
};

// ---- fast filter (no breakdown requested) ---------------------------------
// The decision only needs the SIGN of J - tau.  Utilities from fp32 logs
// (summed in fp64) and tau from an fp32 exp are within a proven bound of the
// exact fp64 values (|du| <= 1e-5, |dtau| <= 1e-4 |tau0 - tau_inf|); when
// |J_fast - tau_fast| exceeds the induced margin the decision is provably the
// exact one, otherwise the row is recomputed exactly (CPython-order fp64).
// Validation (the sum check) is always exact.
__device__ __forceinline__ double entropy_term_fast(double p) {
  const float pf = (float)p;
  return (pf > 0.0f) ? (double)(pf * __logf(pf)) : 0.0;   // p < FLT_MIN: |p ln p| < 1e-36
}

// Returns the decision code, or -1 when J is too close to tau to decide fast.
__device__ __forceinline__ int decide_fast(const AdmitArgs& a, const BatchConst& b, double u_f,
                                           double du, double now) {
  const gg_params& p = a.p;
  const double j = p.alpha * u_f + p.beta * b.e + p.gamma * b.c;
  double el = now - b.t_origin;
  el = (el > 0.0) ? el : 0.0;
  const double e = (double)__expf((float)(-p.k * el));
  const double tau = p.tau_inf + (p.tau0 - p.tau_inf) * e;
  const double margin = fabs(p.alpha) * du + fabs(p.tau0 - p.tau_inf) * 1e-4 + 1e-12;
  if (fabs(j - tau) <= margin) return -1;
  const bool admit = (p.direction == GG_DIR_GEQ) ? (j > tau) : (j < tau);
  if (!admit) return GG_DECISION_SKIP;
  if (p.routing == GG_ROUTE_ALL_BATCHED) return GG_DECISION_BATCHED;
  if (p.routing == GG_ROUTE_THRESHOLD_ON_QUEUE)
    return (b.qd > (int64_t)p.queue_threshold) ? GG_DECISION_BATCHED : GG_DECISION_DIRECT;
  return GG_DECISION_DIRECT;
}

// The per-request tail of decide(): J, tau(now), admit, route
// (controller.py:326-337).
__device__ __forceinline__ uint8_t decide_row(const AdmitArgs& a, const BatchConst& b, double u,
                                              double now, double& j, double& tau) {
  const gg_params& p = a.p;
  j = f64_add(f64_add(f64_mul(p.alpha, u), f64_mul(p.beta, b.e)), f64_mul(p.gamma, b.c));
  double el = f64_sub(now, b.t_origin);
  el = (el > 0.0) ? el : 0.0;
  tau = f64_add(p.tau_inf, f64_mul(f64_sub(p.tau0, p.tau_inf), exp(f64_mul(-p.k, el))));
  bool admit = (p.direction == GG_DIR_GEQ) ? (j >= tau) : (j < tau);
  if (!admit) return GG_DECISION_SKIP;
  if (p.routing == GG_ROUTE_ALL_BATCHED) return GG_DECISION_BATCHED;
  if (p.routing == GG_ROUTE_THRESHOLD_ON_QUEUE)
    return (b.qd > (int64_t)p.queue_threshold) ? GG_DECISION_BATCHED : GG_DECISION_DIRECT;
  return GG_DECISION_DIRECT;
}

template <int THREADS, int RPT>
struct AdmitShared {
  static constexpr int WARPS = THREADS / 32;
  static constexpr int GROUPS = RPT * WARPS;   // 32-row groups, in row order
  BatchConst bc;
  int64_t row0, nw, depth0;   // window start/length; FIFO depth before this launch
  unsigned long long block_prefix;
  int group_cnt[GROUPS];
  int group_off[GROUPS];
  int warp_skip[WARPS];
  int vb;
  int last;
};

__device__ __forceinline__ int warp_sum(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long t = __shfl_xor_sync(0xffffffffu, v, o);
    v = t > v ? t : v;
  }
  return v;
}

// Per-block prologue (thread 0): decision window, FIFO depth and the
// batch-constant E/C — all read before any block can finalize.  Tiles are
// scanned in blockIdx order (blocks are dispatched in increasing linear order,
// so every predecessor of a resident block is resident or finished — the same
// forward-progress argument CUB's single-pass scan relies on), which lets each
// thread issue its row loads before this prologue completes.
template <int THREADS, int RPT>
__device__ void block_setup(const AdmitArgs& a, AdmitShared<THREADS, RPT>& sm) {
  sm.vb = (int)blockIdx.x;
  int64_t row0, nw;
  admit_window(a, row0, nw);
  sm.row0 = row0;
  sm.nw = nw;
  sm.depth0 = a.fifo ? a.fifo->tail - a.fifo->head : 0;
  sm.bc = batch_constants(a.state, a.snap, a.fifo);
}

// Apply one decide_batch's state effects (controller.py:316-337) once, after
// every block has read the state: observes of the frozen snapshot, the
// admitted/skipped totals, the FIFO tail/cursor, the batch info; then leave the
// workspace header zeroed for the next launch.  `counts` = pack_counts(adm, skip).
__device__ void finalize_launch(const AdmitArgs& a, const BatchConst& b, int64_t row0, int64_t nw,
                                int64_t depth0, unsigned long long counts,
                                unsigned long long benc) {
  const int64_t n_adm = (int64_t)(counts & kCnt31);
  const int64_t n_skip = (int64_t)((counts >> 31) & kCnt31);
  const int64_t n_inv = nw - n_adm - n_skip;
  gg_state* st = a.state;
  const bool any_valid = (nw - n_inv) > 0;
  if (any_valid) {
    if (b.samples_seen > 0) ch_observe(st->n_energy, b.ewma);
    ch_observe(st->n_queue_depth, (double)b.qd);
    ch_observe(st->n_p95_ms, b.p95);
  }
  st->admitted_total += n_adm;
  st->skipped_total += n_skip;
  if (a.fifo) {
    const int64_t room = a.fifo->capacity - depth0;
    a.fifo->tail += n_adm < room ? n_adm : room;
    a.fifo->cursor = row0 + nw;
  }
  if (a.info) {
    a.info->n_admitted = n_adm;
    a.info->n_skipped = n_skip;
    a.info->n_invalid = n_inv;
    a.info->first_invalid = benc ? (int64_t)(row0 + nw - (int64_t)benc) : -1;
    a.info->energy = any_valid ? b.e : 0.0;
    a.info->congestion = any_valid ? b.c : 0.0;
    a.info->n_decided = nw;
    a.info->snap_queue_depth = b.qd;
    a.info->snap_p95_ms = b.p95;
    a.info->snap_batch_fill = b.fill;
  }
  a.ws->vblock_counter = 0;
  a.ws->done_counter = 0;
  a.ws->n_skipped = 0;
  a.ws->n_invalid = 0;
  a.ws->first_invalid_enc = 0;
}

// Order-preserving compaction of the tile + counters + last-block finalize.
template <int THREADS, int RPT>
__device__ void finish_tile(const AdmitArgs& a, AdmitShared<THREADS, RPT>& sm, int64_t tile0,
                            const uint32_t (&ballots)[RPT], int my_skip,
                            unsigned long long my_bad_enc) {
  constexpr int WARPS = THREADS / 32;
  constexpr int GROUPS = RPT * WARPS;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ws = warp_sum(my_skip);
  if (lane == 0) {
#pragma unroll
    for (int j = 0; j < RPT; ++j) sm.group_cnt[j * WARPS + warp] = __popc(ballots[j]);
    sm.warp_skip[warp] = ws;
  }
  // first invalid row: rare, one atomic per warp that has one
  if (__any_sync(0xffffffffu, my_bad_enc != 0ull)) {
    const unsigned long long wb = warp_max_u64(my_bad_enc);
    if (lane == 0) atomicMax(&a.ws->first_invalid_enc, wb);
  }
  __syncthreads();
  if (warp == 0) {
    constexpr int GPL = (GROUPS + 31) / 32;   // consecutive groups per lane
    int c[GPL];
    int mine = 0;
#pragma unroll
    for (int q = 0; q < GPL; ++q) {
      const int gi = lane * GPL + q;
      c[q] = gi < GROUPS ? sm.group_cnt[gi] : 0;
      mine += c[q];
    }
    int v = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int t = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += t;
    }
    const int total = __shfl_sync(0xffffffffu, v, 31);
    int run = v - mine;
#pragma unroll
    for (int q = 0; q < GPL; ++q) {
      const int gi = lane * GPL + q;
      if (gi < GROUPS) sm.group_off[gi] = run;
      run += c[q];
    }
    const int skip = warp_sum(lane < WARPS ? sm.warp_skip[lane] : 0);
    const unsigned long long pre = lookback_warp(
        a.ws->status, sm.vb, pack_counts((unsigned long long)total, (unsigned long long)skip));
    if (lane == 0) sm.block_prefix = pre & kCnt31;
  }
  __syncthreads();
  if (a.admitted_idx || a.ring) {
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
      if ((ballots[j] >> lane) & 1u) {
        unsigned long long pos = sm.block_prefix + sm.group_off[j * WARPS + warp] +
                                 __popc(ballots[j] & ((1u << lane) - 1u));
        const int64_t r = tile0 + (int64_t)j * THREADS + tid;
        if (a.admitted_idx) a.admitted_idx[pos] = (int32_t)r;
        if (a.ring) {  // enqueue in trace order behind the current FIFO tail
          const int64_t cap = a.fifo->capacity;
          if (sm.depth0 + (int64_t)pos < cap) {
            const int64_t slot = (a.fifo->tail + (int64_t)pos) & (cap - 1);
            a.ring[slot] = (int32_t)(sm.row0 + r);
            if (a.ring_ns) a.ring_ns[slot] = globaltimer_ns();
          } else {
            atomicAdd(reinterpret_cast<unsigned long long*>(&a.fifo->overflow), 1ull);
          }
        }
      }
    }
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    unsigned long long t = atomicAdd(&a.ws->done_counter, 1ull);
    sm.last = (t == (unsigned long long)gridDim.x - 1ull);
  }
  __syncthreads();
  if (!sm.last) return;
  // ---- last block: every other block has finished reading state and writing
  // its counters; apply the batch's state effects once (controller.py:316-337).
  __threadfence();
  if (tid == 0) {
    const unsigned long long w = ld_relaxed(&a.ws->status[gridDim.x - 1]);
    finalize_launch(a, sm.bc, sm.row0, sm.nw, sm.depth0, w, ld_relaxed(&a.ws->first_invalid_enc));
  }
  __syncthreads();
  for (int i = tid; i < (int)gridDim.x; i += THREADS) a.ws->status[i] = 0ull;
}

// ---- K1, small K (K <= 16) -------------------------------------------------
// Batch-constant part of the single-precision fast filter.  J and tau are
// evaluated in fp32; the margin covers (a) the utility error du of the fp32
// logs, (b) the fp32 exp error (1e-4 relative of |tau0 - tau_inf|) and (c) the
// fp32 rounding of every operand and operation (1e-6 x the operand scale).
// Rows inside the margin (and NaN) are recomputed exactly.
struct FastBlock {
  double t_origin;
  float alpha, jc, tau_inf, dtau, negk_log2e, margin, inv_log2k;
  int geq;
  int adm_code;   // DIRECT / BATCHED: routing depends only on batch constants
};

constexpr int kNeedExact = 255;

__device__ FastBlock fast_block(const AdmitArgs& a, const BatchConst& b) {
  const gg_params& p = a.p;
  FastBlock f;
  f.t_origin = b.t_origin;
  const double jc = p.beta * b.e + p.gamma * b.c;
  f.alpha = (float)p.alpha;
  f.jc = (float)jc;
  f.tau_inf = (float)p.tau_inf;
  f.dtau = (float)(p.tau0 - p.tau_inf);
  f.negk_log2e = (float)(-p.k * 1.4426950408889634);
  f.inv_log2k = (float)(0.6931471805599453 / a.ln_k);
  const double scale = fabs(p.alpha) + fabs(jc) + fabs(p.tau0) + fabs(p.tau_inf) + 1.0;
  const double du = (p.utility_proxy == GG_UTIL_ENTROPY) ? 1e-5 : 0.0;
  const double m = fabs(p.alpha) * du + fabs(p.tau0 - p.tau_inf) * 1e-4 + 1e-6 * scale;
  f.margin = (scale < 1e30) ? (float)m : INFINITY;   // out of fp32 range: always exact
  f.geq = p.direction == GG_DIR_GEQ;
  if (p.routing == GG_ROUTE_ALL_BATCHED) f.adm_code = GG_DECISION_BATCHED;
  else if (p.routing == GG_ROUTE_THRESHOLD_ON_QUEUE)
    f.adm_code = (b.qd > (int64_t)p.queue_threshold) ? GG_DECISION_BATCHED : GG_DECISION_DIRECT;
  else f.adm_code = GG_DECISION_DIRECT;
  return f;
}

// Fast decision for one row: exact validation (_validate_distribution,
// controller.py:126-136), fp32 utility, fp32 J - tau, margin test.  Returns a
// decision code or kNeedExact.  K <= 4 sums the fp32 entropy terms in fp32
// (|du| <= K (4e-7 + 6e-8) / ln 2 < 1e-5); the generic K <= 16 path in fp64.
// tau's exp runs as ex2.approx of a pre-scaled argument: relative error
// <= 2^-22 + 1.8e-7 |k el| (argument rounding), inside the 1e-4 allowance
// wherever exp(-k el) > 2^-30, and negligible in absolute terms elsewhere.
__device__ __forceinline__ float lg2_approx(float x) {   // MUFU.LG2, denormals flushed
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float ex2_approx(float x) {   // MUFU.EX2
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <int KC>
__device__ __forceinline__ int fast_row(const double* x, int k, double now, const FastBlock& f,
                                        bool entropy) {
  bool ok = true, first = true;
  double mx = 0.0, hd = 0.0, tot;
  float hf = 0.0f;
  NeumaierSum ns;
#pragma unroll
  for (int c = 0; c < (KC > 0 ? KC : 16); ++c) {
    if (KC == 0 && c >= k) break;
    const double xc = x[c];
    // finite and >= 0.  K = 2: x >= 0 alone suffices -- NaN fails it, and an
    // infinite value (the other one >= 0) makes the total inf, failing the sum check
    ok = ok && (xc >= 0.0) && (KC == 2 || xc <= 1.7976931348623157e308);
    if (KC != 2) ns.add(xc);
    if (entropy) {   // p log2 p; u = -sum / log2 K (the ln 2 factors cancel)
      const float pf = (float)xc;
      const float t = pf > 0.0f ? pf * lg2_approx(pf) : 0.0f;
      if (KC > 0) hf += t;
      else hd += (double)t;
    } else {
      mx = (first || xc > mx) ? xc : mx;
      first = false;
    }
  }
  // K = 2: Neumaier's sum of [x0, x1] is t + c with c the exact error of
  // t = fl(x0 + x1), and fl(t + c) == t — the validation total is one add.
  if constexpr (KC == 2) tot = f64_add(x[0], x[1]);
  else tot = ns.result();
  if (!ok || k < 2 || fabs(f64_sub(tot, 1.0)) > 1e-9) return GG_DECISION_INVALID;
  float u;
  if (entropy) u = fminf(fmaxf(-(KC > 0 ? hf : (float)hd) * f.inv_log2k, 0.0f), 1.0f);
  else u = (float)(1.0 - mx);
  const float el = fmaxf((float)(now - f.t_origin), 0.0f);   // == (float)fmax(now - t0, 0.0)
  const float tau = f.tau_inf + f.dtau * ex2_approx(f.negk_log2e * el);
  const float d = (f.alpha * u + f.jc) - tau;
  if (!(fabsf(d) > f.margin)) return kNeedExact;
  return (f.geq ? d > 0.0f : d < 0.0f) ? f.adm_code : GG_DECISION_SKIP;
}

// The reference's own evaluation of one row (CPython order, fp64).
__device__ __forceinline__ int exact_row(const AdmitArgs& a, const BatchConst& b, const double* row,
                                         int k, double now, bool entropy, double* bd3) {
  RowAcc acc;   // controller.py:126-148
  for (int c = 0; c < k; ++c) acc.add(row[c], entropy);
  double u, jv = 0.0, tau = 0.0;
  int code;
  if (acc.finish(k, entropy, a.ln_k, u)) {
    code = decide_row(a, b, u, now, jv, tau);
  } else {
    code = GG_DECISION_INVALID;
    u = jv = tau = __longlong_as_double(0x7ff8000000000000ll);
  }
  if (bd3) {
    bd3[0] = u;
    bd3[1] = jv;
    bd3[2] = tau;
  }
  return code;
}

// RPT rows per thread (row = tile0 + j*256 + tid: a warp's rows are contiguous,
// so its loads of a [32 x K] fp64 slab coalesce).  K = 2, 4: all RPT rows and
// arrival times are loaded into registers before anything else.
// BD: breakdown requested -> every row takes the exact path.
// SPLIT: large batches — the batch constants come precomputed from
// admit_prologue_kernel (no per-block prologue, no barrier before the rows),
// and the kernel only decides + writes per-block counts (and their super-block
// sums); admit_compact_kernel finishes (no cross-block waiting anywhere).
constexpr int kSmallThreads = 256;

struct SplitConsts {
  BatchConst bc;
  FastBlock fb;
};
static_assert(sizeof(SplitConsts) <= sizeof(((AdmitWorkspace*)0)->consts), "workspace consts");

// UP: the utility proxy as a compile-time constant on the fast path (1 entropy,
// 2 one-minus-confidence; 0 = read at run time) -- the per-row proxy branch was a
// quarter of the decide kernel's instructions.
template <int KC, int RPT, bool BD, bool SPLIT, int UP = 0>
__global__ void __launch_bounds__(kSmallThreads) admit_small_kernel(AdmitArgs a) {
  griddep_wait();   // PDL: the predecessor has completed and flushed
  griddep_launch();
  constexpr int THREADS = kSmallThreads;
  __shared__ AdmitShared<THREADS, RPT> sm;
  __shared__ FastBlock fb_s;
  const int tid = threadIdx.x;
  int64_t row0, nw;
  admit_window(a, row0, nw);
  const int64_t tile0 = (int64_t)blockIdx.x * THREADS * RPT;
  // rows of this thread: j*THREADS < rem  (32-bit compares; pointers stepped)
  const int64_t rem64 = nw - tile0 - tid;
  const int rem = rem64 > THREADS * RPT ? THREADS * RPT : (int)rem64;
  const int64_t g0 = row0 + tile0 + tid;   // trace row of j = 0
  constexpr bool PRE = KC > 0 && !BD;
  double px[PRE ? RPT : 1][KC > 0 ? KC : 2], pn[PRE ? RPT : 1];
  if constexpr (PRE) {
    const double* rp = a.probs + g0 * a.stride;
    const double* np = a.now + g0;
    const int64_t step = (int64_t)THREADS * a.stride;
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
      if (j * THREADS < rem) {
#pragma unroll
        for (int c = 0; c < KC; c += 2) {
          const double2 v = __ldg(reinterpret_cast<const double2*>(rp + c));
          px[j][c] = v.x;
          px[j][c + 1] = v.y;
        }
        pn[j] = __ldg(np);
      }
      rp += step;
      np += THREADS;
    }
  }
  const SplitConsts* sc = reinterpret_cast<const SplitConsts*>(a.ws->consts);
  if constexpr (!SPLIT) {
    if (tid == 0) {
      block_setup(a, sm);
      fb_s = fast_block(a, sm.bc);
    }
    __syncthreads();
  }
  const bool entropy = UP == 0 ? a.p.utility_proxy == GG_UTIL_ENTROPY : UP == 1;
  const int k = KC > 0 ? KC : a.k;
  int code[RPT];
  bool any_exact = false;
  if constexpr (!BD) {
    const FastBlock f = SPLIT ? sc->fb : fb_s;
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
      int c = GG_DECISION_SKIP;
      if (j * THREADS < rem) {
        if constexpr (KC > 0) {
          c = fast_row<KC>(px[j], k, pn[j], f, entropy);
        } else {
          const int64_t g = g0 + (int64_t)j * THREADS;
          const double* row = a.probs + g * a.stride;
          double xv[16];
#pragma unroll
          for (int q = 0; q < 16; ++q) xv[q] = q < k ? row[q] : 0.0;
          c = fast_row<0>(xv, k, a.now[g], f, entropy);
        }
      }
      code[j] = c;
      any_exact |= (c == kNeedExact);
    }
  }
  if (BD || __any_sync(0xffffffffu, any_exact)) {   // rare without a breakdown
    const BatchConst b = SPLIT ? sc->bc : sm.bc;
#pragma unroll 1
    for (int j = 0; j < RPT; ++j) {
      if (j * THREADS < rem && (BD || code[j] == kNeedExact)) {
        const int64_t g = g0 + (int64_t)j * THREADS;
        code[j] = exact_row(a, b, a.probs + g * a.stride, k, a.now[g], entropy,
                            BD && a.breakdown ? a.breakdown + 3 * g : nullptr);
      } else if (BD) {
        code[j] = GG_DECISION_SKIP;
      }
    }
  }
  uint32_t ballots[RPT];
  int my_skip = 0;
  int first_bad = -1;
  uint8_t* dp = a.decision + g0;
#pragma unroll
  for (int j = 0; j < RPT; ++j) {
    const bool in = j * THREADS < rem;
    if (in) {
      dp[j * THREADS] = (uint8_t)code[j];
      my_skip += code[j] == GG_DECISION_SKIP;
      if (code[j] == GG_DECISION_INVALID && first_bad < 0) first_bad = j;
    }
    ballots[j] = __ballot_sync(0xffffffffu, in && (code[j] == GG_DECISION_DIRECT || code[j] == GG_DECISION_BATCHED));
  }
  const unsigned long long my_bad =
      first_bad < 0 ? 0ull : (unsigned long long)(rem64 - (int64_t)first_bad * THREADS);   // nw - r
  if constexpr (SPLIT) {
    constexpr int WARPS = THREADS / 32;
    const int lane = tid & 31, warp = tid >> 5;
    int wa = 0;
#pragma unroll
    for (int j = 0; j < RPT; ++j) wa += __popc(ballots[j]);
    const int ws = warp_sum(my_skip);
    if (lane == 0) {
      sm.group_cnt[warp] = wa;
      sm.warp_skip[warp] = ws;
    }
    if (__any_sync(0xffffffffu, my_bad != 0ull)) {
      const unsigned long long wb = warp_max_u64(my_bad);
      if (lane == 0) atomicMax(&a.ws->first_invalid_enc, wb);
    }
    __syncthreads();
    if (warp == 0) {
      const int adm = warp_sum(lane < WARPS ? sm.group_cnt[lane] : 0);
      const int skp = warp_sum(lane < WARPS ? sm.warp_skip[lane] : 0);
      if (lane == 0) {
        const unsigned long long pc = pack_counts((unsigned long long)adm, (unsigned long long)skp);
        a.split_cnt[blockIdx.x] = pc;
        atomicAdd(&a.super_cnt[blockIdx.x >> a.super_shift], pc);
      }
    }
  } else {
    finish_tile<THREADS, RPT>(a, sm, tile0, ballots, my_skip, my_bad);
  }
}

// SPLIT step 0 (one thread): the launch's batch constants, once.
__global__ void admit_prologue_kernel(AdmitArgs a) {
  griddep_wait();   // PDL: the predecessor has completed and flushed
  griddep_launch();
  if (threadIdx.x != 0) return;
  SplitConsts* sc = reinterpret_cast<SplitConsts*>(a.ws->consts);
  const BatchConst b = batch_constants(a.state, a.snap, nullptr);
  sc->bc = b;
  sc->fb = fast_block(a, b);
}

// SPLIT step 2: order-preserving compaction from the decision bytes.  A block
// owns 8192 rows (= 4 decide tiles); its global offset is the sum of the super-
// block counts before it plus the decide-block counts inside its super-block
// (<= 2 sqrt(#blocks) words, no scan launch, no waiting).  Each lane turns 32
// consecutive decision bytes (two 16-B loads) into a bit mask; admitted row
// ids are staged in shared memory in order and written out coalesced.  The
// last block to finish applies the launch's state effects and re-zeroes the
// split counters.
constexpr int kCompactRows = 8192;
constexpr int kDecideRows = kSmallThreads * 8;   // decide tile (kSmallRpt rows per thread)

__global__ void __launch_bounds__(kSmallThreads) admit_compact_kernel(AdmitArgs a, int nb_decide) {
  griddep_wait();   // PDL: the predecessor has completed and flushed
  griddep_launch();
  constexpr int THREADS = kSmallThreads, WARPS = THREADS / 32;
  __shared__ int32_t out[kCompactRows];
  __shared__ int warp_off[WARPS];
  __shared__ unsigned long long red[WARPS];
  __shared__ int last, tot_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t c0 = (int64_t)blockIdx.x * kCompactRows;
  // ---- masks of admitted rows: lane owns rows r0 .. r0+31.  The decision loads
  // are issued first so their latency overlaps the prefix loads below.
  const int64_t r0 = c0 + (int64_t)(warp * 32 + lane) * 32;
  uint32_t mask = 0;
  const bool vec = ((reinterpret_cast<uintptr_t>(a.decision) & 15) == 0) && r0 + 32 <= a.n;
  uint4 u0 = make_uint4(0, 0, 0, 0), u1 = u0;
  if (vec) {
    const uint4* p4 = reinterpret_cast<const uint4*>(a.decision + r0);
    u0 = __ldcs(p4);
    u1 = __ldcs(p4 + 1);
  }
  // ---- global offset of this block: decide block i0 = first of its tiles
  const int i0 = (int)(c0 / kDecideRows);
  const int sup = i0 >> a.super_shift, sup0 = sup << a.super_shift;
  unsigned long long part = 0;
  for (int q = tid; q < sup + (i0 - sup0); q += THREADS)
    part += q < sup ? a.super_cnt[q] : a.split_cnt[sup0 + (q - sup)];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  if (lane == 0) red[warp] = part;
  if (vec) {
    const uint32_t w[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
#pragma unroll
    for (int q = 0; q < 8; ++q) {
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const uint32_t c = (w[q] >> (8 * b)) & 0xFFu;
        mask |= (uint32_t)(c == GG_DECISION_DIRECT || c == GG_DECISION_BATCHED) << (q * 4 + b);
      }
    }
  } else {
    for (int i = 0; i < 32; ++i) {
      if (r0 + i < a.n) {
        const int c = a.decision[r0 + i];
        mask |= (uint32_t)(c == GG_DECISION_DIRECT || c == GG_DECISION_BATCHED) << i;
      }
    }
  }
  const int cnt = __popc(mask);
  int v = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  if (lane == 31) warp_off[warp] = v;
  __syncthreads();
  if (warp == 0) {
    const int w = lane < WARPS ? warp_off[lane] : 0;
    int x = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += t;
    }
    if (lane < WARPS) warp_off[lane] = x - w;
  }
  __syncthreads();
  unsigned long long base = 0;
#pragma unroll
  for (int q = 0; q < WARPS; ++q) base += red[q];
  int pos = warp_off[warp] + (v - cnt);
  for (uint32_t m = mask; m; m &= m - 1) out[pos++] = (int32_t)(r0 + __ffs(m) - 1);
  // block total = last warp's offset + its inclusive sum (broadcast via smem)
  if (warp == WARPS - 1 && lane == 31) tot_s = warp_off[warp] + v;
  // ---- completion count: every block has consumed its prefix words (split /
  // super counts) before it counts itself done, and nothing the last block
  // reads is written by this kernel, so no fence over the index stores below
  // (a __threadfence there held each block until its stores were acknowledged)
  if (tid == 0) last = atomicAdd(&a.ws->done_counter, 1ull) == (unsigned long long)gridDim.x - 1ull;
  __syncthreads();
  if (a.admitted_idx) {
    int32_t* dst = a.admitted_idx + (base & kCnt31);
    for (int i = tid; i < tot_s; i += THREADS) __stcs(dst + i, out[i]);
  }
  if (!last) return;
  __threadfence();
  const int nsup = ((nb_decide - 1) >> a.super_shift) + 1;
  unsigned long long tot = 0;
  for (int q = tid; q < nsup; q += THREADS) tot += a.super_cnt[q];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
  __syncthreads();
  if (lane == 0) red[warp] = tot;
  __syncthreads();
  if (tid == 0) {
    unsigned long long grand = 0;
    for (int q = 0; q < WARPS; ++q) grand += red[q];
    const BatchConst b = reinterpret_cast<const SplitConsts*>(a.ws->consts)->bc;
    finalize_launch(a, b, 0, a.n, 0, grand, a.ws->first_invalid_enc);
  }
  for (int q = tid; q < nb_decide; q += THREADS) a.split_cnt[q] = 0ull;
  for (int q = tid; q < nsup; q += THREADS) a.super_cnt[q] = 0ull;
}

// K1, large K (ResNet K=1000).  The CPython sums are sequential per row, but
// the K logs are independent, so a block owns 32 rows and splits the work:
//   warps 2..7  stream [32 x 32] column chunks in with coalesced loads and
//               compute p*log(p) for every element (FP64-throughput bound,
//               spread over many SMs instead of one thread per row);
//   warp 0      lane r: Neumaier entropy sum of row r over the precomputed terms
//   warp 1      lane r: validation (finite, >= 0), Neumaier total, max
// double-buffered through shared memory with named barriers, so the two
// sequential chains overlap the log computation of the next chunk.
constexpr int kLargeThreads = 256;
constexpr int kSmallRpt = 8;   // admit_small_kernel rows per thread (2048 rows per block)
constexpr int kLargeRows = 32;
constexpr int kChunk = 32;
constexpr int kProdThreads = kLargeThreads - 64;

__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__global__ void __launch_bounds__(kLargeThreads) admit_large_kernel(AdmitArgs a) {
  griddep_wait();   // PDL: the predecessor has completed and flushed
  griddep_launch();
  __shared__ AdmitShared<kLargeThreads, 1> sm;
  __shared__ double raw[2][kLargeRows][kChunk + 1];
  __shared__ double term[2][kLargeRows][kChunk + 1];
  __shared__ double tot_s[kLargeRows], max_s[kLargeRows];
  __shared__ int ok_s[kLargeRows];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) block_setup(a, sm);
  __syncthreads();
  const BatchConst b = sm.bc;
  const int64_t tile0 = (int64_t)sm.vb * kLargeRows;
  const int64_t nw = sm.nw, row0 = sm.row0;
  const bool entropy = a.p.utility_proxy == GG_UTIL_ENTROPY;
  const int nchunks = (a.k + kChunk - 1) / kChunk;
  // named barriers: 1,2 = buffer full; 3,4 = buffer free
  if (warp >= 2) {
    const int pt = tid - 64;
    for (int c = 0; c < nchunks; ++c) {
      const int buf = c & 1, c0 = c * kChunk, cw = min(kChunk, a.k - c0);
      if (c >= 2) named_sync(3 + buf, kLargeThreads);
      for (int e = pt; e < kLargeRows * kChunk; e += kProdThreads) {
        const int rr = e / kChunk, cc = e % kChunk;
        const int64_t lr = tile0 + rr;
        double v = 0.0, t = 0.0;
        if (lr < nw && cc < cw) {
          v = __ldg(a.probs + (row0 + lr) * a.stride + c0 + cc);
          if (entropy && v > 0.0) t = f64_mul(v, log(v));
        }
        raw[buf][rr][cc] = v;
        term[buf][rr][cc] = t;
      }
      named_arrive(1 + buf, kLargeThreads);
    }
  } else {
    NeumaierSum s;   // warp 0: entropy terms; warp 1: the validation total
    bool ok = true, first = true;
    double mx = 0.0;
    for (int c = 0; c < nchunks; ++c) {
      const int buf = c & 1, cw = min(kChunk, a.k - c * kChunk);
      named_sync(1 + buf, kLargeThreads);
      // unrolled with a guard so the shared-memory loads issue ahead of the
      // loop-carried Neumaier chain
      if (warp == 0) {
        if (entropy) {
#pragma unroll 8
          for (int cc = 0; cc < kChunk; ++cc)
            if (cc < cw && raw[buf][lane][cc] > 0.0) s.add(term[buf][lane][cc]);
        }
      } else {
#pragma unroll 8
        for (int cc = 0; cc < kChunk; ++cc) {
          if (cc >= cw) break;
          const double x = raw[buf][lane][cc];
          if (!isfinite(x) || x < 0.0) ok = false;
          s.add(x);
          if (first || x > mx) mx = x;
          first = false;
        }
      }
      if (c + 2 < nchunks) named_arrive(3 + buf, kLargeThreads);
    }
    if (warp == 1) {
      tot_s[lane] = s.result();
      ok_s[lane] = ok;
      max_s[lane] = mx;
    }
    named_sync(5, 64);
    if (warp == 0) {
      // fold the two chains into the RowAcc::finish logic (controller.py:126-148)
      const bool valid = ok_s[lane] && a.k >= 2 && !(fabs(f64_sub(tot_s[lane], 1.0)) > 1e-9);
      double u = 0.0;
      if (valid) u = entropy ? clamp01(f64_div(-s.result(), a.ln_k)) : f64_sub(1.0, max_s[lane]);
      tot_s[lane] = u;
      ok_s[lane] = valid;
    }
  }
  __syncthreads();
  const int64_t r = tile0 + tid;           // rows live on warp 0's lanes
  const bool in = warp == 0 && r < nw;
  const int64_t g = row0 + r;
  uint8_t code = GG_DECISION_SKIP;
  int my_skip = 0;
  unsigned long long my_bad = 0;
  if (in) {
    double u = tot_s[lane], jv = 0.0, tau = 0.0;
    if (ok_s[lane]) {
      code = decide_row(a, b, u, a.now[g], jv, tau);
      if (code == GG_DECISION_SKIP) ++my_skip;
    } else {
      code = GG_DECISION_INVALID;
      if (!my_bad) my_bad = (unsigned long long)(nw - r);
      u = jv = tau = __longlong_as_double(0x7ff8000000000000ll);
    }
    a.decision[g] = code;
    if (a.breakdown) {
      a.breakdown[3 * g] = u;
      a.breakdown[3 * g + 1] = jv;
      a.breakdown[3 * g + 2] = tau;
    }
  }
  uint32_t ballots[1] = {__ballot_sync(0xffffffffu, in && (code == GG_DECISION_DIRECT || code == GG_DECISION_BATCHED))};
  finish_tile<kLargeThreads, 1>(a, sm, tile0, ballots, my_skip, my_bad);
}

// K1, large K, fast filter (no breakdown requested; the serving loop): one warp
// per row (16 warps x 2 rows, 32 rows per block), coalesced loads, fp64 sum of the
// probabilities and of fp32-log entropy terms, warp reductions — no sequential
// chain.  For K <= 1024 a row is preloaded into registers (all loads in flight
// at once: a small serving window is latency-, not bandwidth-bound).  A row is
// recomputed exactly — in CPython order — only when its sum lies within 1e-13
// of the 1e-9 validation bound or J lies within the margin of tau; the exact
// fp64 logs are then computed lane-parallel and only the Neumaier chains run
// in element order (every lane evaluates them redundantly, via shuffles).
// Exact (CPython-order) evaluation of one large-K row by a whole warp: the fp64
// logs are computed lane-parallel, 32 elements at a time, and the Neumaier
// chains consume them in element order via shuffles (every lane evaluates the
// chains redundantly).  Compact loop, kept out of line: it is the cold path.
__device__ __noinline__ int exact_row_warp(const AdmitArgs& a, const BatchConst& b,
                                           const double* row, int k, double now, bool entropy,
                                           double mx) {
  const int lane = threadIdx.x & 31;
  NeumaierSum tot, h;
  bool okx = true;
#pragma unroll 1
  for (int c0 = 0; c0 < k; c0 += 32) {
    const int c = c0 + lane;
    const double x = c < k ? row[c] : 0.0;
    const double t = (entropy && x > 0.0) ? f64_mul(x, log(x)) : 0.0;
    const int cnt = min(32, k - c0);
#pragma unroll 1
    for (int j = 0; j < cnt; ++j) {   // element c0 + j, in order
      const double xj = __shfl_sync(0xffffffffu, x, j);
      const double tj = __shfl_sync(0xffffffffu, t, j);
      if (!isfinite(xj) || xj < 0.0) okx = false;
      tot.add(xj);
      if (entropy && xj > 0.0) h.add(tj);
    }
  }
  // RowAcc::finish (controller.py:126-148); max is order-independent
  const bool v = okx && k >= 2 && !(fabs(f64_sub(tot.result(), 1.0)) > 1e-9);
  if (!v) return GG_DECISION_INVALID;
  const double u = entropy ? clamp01(f64_div(-h.result(), a.ln_k)) : f64_sub(1.0, mx);
  double jv, tau;
  return decide_row(a, b, u, now, jv, tau);
}

constexpr int kFastRows = 8;                 // rows per block: one warp per row
constexpr int kFastThreads = 32 * kFastRows;
constexpr int kRegChunks = 32;               // K <= 32 * 32: the row is loaded in one go

// Finite and >= 0 (including -0.0), from the bits: one 64-bit compare.
__device__ __forceinline__ bool finite_nonneg(double x) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(x);
  return u < 0x7FF0000000000000ull || u == 0x8000000000000000ull;
}

template <bool REG>
__global__ void __launch_bounds__(kFastThreads) admit_large_fast_kernel(AdmitArgs a) {
#ifdef GG_K1_PROF
  const unsigned long long tp0 = globaltimer_ns();
#endif
  griddep_wait();   // PDL: the predecessor has completed and flushed
  griddep_launch();
#ifdef GG_K1_PROF
  const unsigned long long tp1 = globaltimer_ns();
#endif
  __shared__ AdmitShared<kFastThreads, 1> sm;
  __shared__ FastBlock fb_s;
  __shared__ uint8_t codes[kFastRows];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  int64_t row0, nw;
  admit_window(a, row0, nw);
  const int64_t tile0 = (int64_t)blockIdx.x * kFastRows;
  const int64_t r = tile0 + warp;                // this warp's row
  const bool have = r < nw;
  const int k = a.k;
  const double* row = a.probs + (row0 + (have ? r : 0)) * a.stride;
  double xr[REG ? kRegChunks : 1];
  if constexpr (REG) {   // all loads in flight before the prologue
#pragma unroll
    for (int i = 0; i < kRegChunks; ++i) {
      const int c = i * 32 + lane;
      xr[i] = (have && c < k) ? __ldg(row + c) : 0.0;
    }
  }
  // the row's arrival time too (the decision needs it right after the reductions)
  const double now_g = have ? __ldg(a.now + row0 + r) : 0.0;
  if (tid == 0) {
    block_setup(a, sm);
    fb_s = fast_block(a, sm.bc);
  }
  __syncthreads();
#ifdef GG_K1_PROF
  const unsigned long long tp2 = globaltimer_ns();
#endif
  const bool entropy = a.p.utility_proxy == GG_UTIL_ENTROPY;
  if (have) {
    const int64_t g = row0 + r;
    double sum = 0.0, mx = -INFINITY;
    float hf = 0.0f;   // per-lane fp32 partial of sum p log2 p (<= 32 terms)
    bool ok = true;
    auto take = [&](double x) {
      ok &= finite_nonneg(x);
      sum += x;
      if (entropy) {
        const float pf = (float)x;
        hf += pf > 0.0f ? pf * lg2_approx(pf) : 0.0f;
      } else {
        mx = fmax(mx, x);
      }
    };
    if constexpr (REG) {
#pragma unroll
      for (int i = 0; i < kRegChunks; ++i)
        if (i * 32 + lane < k) take(xr[i]);
    } else {
      for (int c = lane; c < k; c += 32) take(__ldg(row + c));
    }
    double hd = (double)hf;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      sum += __shfl_xor_sync(0xffffffffu, sum, o);
      hd += __shfl_xor_sync(0xffffffffu, hd, o);
      mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    ok = __all_sync(0xffffffffu, ok);
    // fp64 sum of <= K nonnegative terms: |error| < K * 2^-52 * sum
    const double dev = fabs(sum - 1.0), bound = (double)k * 2.3e-16 * (sum + 1.0);
    int code = GG_DECISION_INVALID;
    bool exact = false, valid = ok && k >= 2;
    if (valid && dev > 1e-9 + bound) valid = false;
    else if (valid && dev > 1e-9 - bound) exact = true;   // too close to the bound
    if (valid && !exact) {
      // fp32 decision as in fast_row; the lane partials add |du| <= 32 * 2^-24 * H2 / log2 K
      // + the lg2.approx error, inside the 1e-5 allowance
      const FastBlock f = fb_s;
      const float u = entropy ? fminf(fmaxf(-(float)hd * f.inv_log2k, 0.0f), 1.0f)
                              : (float)(1.0 - mx);
      const float el = (float)fmax(now_g - f.t_origin, 0.0);
      const float tau = f.tau_inf + f.dtau * ex2_approx(f.negk_log2e * el);
      const float d = (f.alpha * u + f.jc) - tau;
      if (!(fabsf(d) > f.margin)) exact = true;
      else code = (f.geq ? d > 0.0f : d < 0.0f) ? f.adm_code : GG_DECISION_SKIP;
    }
    if (exact)   // warp-uniform; rare: the reference's own evaluation order
      code = exact_row_warp(a, sm.bc, row, k, now_g, entropy, mx);
    if (lane == 0) {
      codes[warp] = (uint8_t)code;
      a.decision[g] = (uint8_t)code;
    }
  }
  __syncthreads();
  // compaction: the block's rows on warp 0's lanes 0..kFastRows-1
  const int64_t rr = tile0 + tid;
  const bool in = warp == 0 && lane < kFastRows && rr < nw;
  const uint8_t code = in ? codes[lane] : (uint8_t)GG_DECISION_SKIP;
  const int my_skip = (in && code == GG_DECISION_SKIP) ? 1 : 0;
  const unsigned long long my_bad =
      (in && code == GG_DECISION_INVALID) ? (unsigned long long)(nw - rr) : 0ull;
  uint32_t ballots[1] = {__ballot_sync(0xffffffffu, in && (code == GG_DECISION_DIRECT || code == GG_DECISION_BATCHED))};
#ifdef GG_K1_PROF
  const unsigned long long tp3 = globaltimer_ns();
#endif
  finish_tile<kFastThreads, 1>(a, sm, tile0, ballots, my_skip, my_bad);
#ifdef GG_K1_PROF
  if (tid == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1))
    printf("K1 block %d/%d: wait %llu, setup+loads %llu, rows %llu, finish %llu ns (start %llu)\n", blockIdx.x,
           gridDim.x, tp1 - tp0, tp2 - tp1, tp3 - tp2, globaltimer_ns() - tp3, tp0 % 1000000ull);
#endif
}

// ---------------------------------------------------------------------------
// K2: record_outcome() x n, sequential in completion order (controller.py:345-358).
// One warp: scalars are evaluated redundantly by every lane (identical values);
// the sorted latency window lives in registers (position i = slot j * 32 +
// lane) and is updated with warp shuffles, so an append/evict plus the
// nearest-rank p95 (telemetry.py:35-46) is a few dozen instructions.

template <int S>  // slots per lane: window capacity 32 * S
struct RegSorted {
  double v[S];
  __device__ __forceinline__ void load(const double* src, int count) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int j = 0; j < S; ++j) {
      const int i = j * 32 + lane;
      v[j] = i < count ? src[i] : INFINITY;
    }
  }
  __device__ __forceinline__ void store(double* dst, int count) const {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int j = 0; j < S; ++j)
      if (j * 32 + lane < count) dst[j * 32 + lane] = v[j];
  }
  __device__ __forceinline__ int count_less(double x) const {
    int c = 0;
#pragma unroll
    for (int j = 0; j < S; ++j) c += __popc(__ballot_sync(0xffffffffu, v[j] < x));
    return c;
  }
  __device__ __forceinline__ int find(double x, int count) const {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int j = 0; j < S; ++j) {
      const unsigned m = __ballot_sync(0xffffffffu, j * 32 + lane < count && v[j] == x);
      if (m) return j * 32 + __ffs(m) - 1;
    }
    return -1;
  }
  __device__ __forceinline__ double at(int i) const {
    double r = 0.0;
#pragma unroll
    for (int j = 0; j < S; ++j)
      if (j == (i >> 5)) r = v[j];
    return __shfl_sync(0xffffffffu, r, i & 31);
  }
  // positions >= pos move up by one, x lands at pos (positions descending so
  // lane 0 still sees the old last element of the previous slot)
  __device__ __forceinline__ void insert_at(int pos, double x) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int j = S - 1; j >= 0; --j) {
      const double up = __shfl_up_sync(0xffffffffu, v[j], 1);
      const double carry = j > 0 ? __shfl_sync(0xffffffffu, v[j > 0 ? j - 1 : 0], 31) : 0.0;
      const int i = j * 32 + lane;
      const double nv = lane == 0 ? carry : up;
      if (i > pos) v[j] = nv;
      else if (i == pos) v[j] = x;
    }
  }
  // positions > pos move down by one; the freed last position becomes +inf
  __device__ __forceinline__ void remove_at(int pos) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int j = 0; j < S; ++j) {
      const double down = __shfl_down_sync(0xffffffffu, v[j], 1);
      const double carry = j + 1 < S ? __shfl_sync(0xffffffffu, v[j + 1 < S ? j + 1 : j], 0) : INFINITY;
      const int i = j * 32 + lane;
      if (i >= pos) v[j] = lane == 31 ? carry : down;
    }
  }
};

// Outcomes come either from three arrays (n of them) or from G exchange slots
// (fp64 GG_SLOT_LEN(B) each, see greengate_b200.h), applied slot by slot in
// rank order.
template <int S>
__device__ __noinline__ void outcome_seq(const gg_params& p, gg_state* st, const double* lat, const double* jou,
                            const int32_t* qd, int64_t n, int set_qd, int64_t* err,
                            const double* slots, int G, int B, int rank, gg_fifo* fifo) {
  __shared__ double win[GG_P95_WINDOW_MAX];
  const int lane = threadIdx.x;
  const int cap = p.p95_window;
  int count = st->win_count, head = st->win_head;
  for (int i = lane; i < cap; i += 32) win[i] = st->win[i];
  RegSorted<S> srt;
  srt.load(st->win_sorted, count);
  double ewma = st->ewma_joules_per_request, total = st->total_joules, p95 = st->p95_current;
  int64_t seen = st->samples_seen, outc = st->outcomes_total;
  gg_channel ce = st->n_energy, cq = st->n_queue_depth, cp = st->n_p95_ms;
  int last_qd = st->queue_depth;
  const double lam = p.ewma_lambda, one_minus_lam = f64_sub(1.0, p.ewma_lambda);
  int64_t bad = -1;
  __syncwarp();
  int64_t adm_other = 0, skip_other = 0;
  if (slots) {
    // Phase 1: the other ranks' admission effects of this step (their decide()
    // observes of their own snapshots and their counters).  min/max observes and
    // sums commute, and nothing read them since admission, so applying them
    // here gives every replica the same state.
    for (int gi = 0; gi < G; ++gi) {
      if (gi == rank) continue;
      const double* sl = slots + (int64_t)gi * (3 * B + 8) + 3 * B;
      if (sl[2] - sl[3] > 0.0) {
        if (seen > 0) ch_observe(ce, ewma);
        ch_observe(cq, sl[6]);
        ch_observe(cp, sl[7]);
      }
      adm_other += (int64_t)sl[4];
      skip_other += (int64_t)sl[5];
    }
  }
  // Inputs are staged through shared memory in chunks (coalesced, all lanes) so
  // the sequential loop never waits on a global-memory round trip.
  constexpr int kStage = 256;
  __shared__ double st_l[kStage], st_j[kStage];
  __shared__ int32_t st_q[kStage];
  const int nslots = slots ? G : 1;
  for (int gi = 0; gi < nslots && bad < 0; ++gi) {
  const double* sl = slots ? slots + (int64_t)gi * (3 * B + 8) : nullptr;
  const int64_t ng = sl ? (int64_t)sl[3 * B] : n;
  for (int64_t i0 = 0; i0 < ng && bad < 0; i0 += kStage) {
  const int cn = (int)min((int64_t)kStage, ng - i0);
  __syncwarp();
  for (int e = lane; e < cn; e += 32) {
    const int64_t i = i0 + e;
    st_l[e] = sl ? sl[i] : lat[i];
    st_j[e] = sl ? sl[B + i] : jou[i];
    st_q[e] = sl ? (int32_t)sl[2 * B + i] : qd[i];
  }
  __syncwarp();
  for (int e = 0; e < cn; ++e) {
    const int64_t i = i0 + e;
    const double L = st_l[e];
    const double J = st_j[e];
    const int32_t Q = st_q[e];
    if (L < 0.0 || J < 0.0 || Q < 0) {  // NegativeMeasurement (controller.py:347-353)
      bad = sl ? (int64_t)gi * B + i : i;
      break;
    }
    // EnergyLedger.observe_request -> ewma_update (energy.py:24-36, 75-87)
    ewma = (seen > 0) ? f64_add(f64_mul(lam, ewma), f64_mul(one_minus_lam, J)) : J;
    seen += 1;
    total = f64_add(total, J);
    // deque(maxlen=p95_window).append(latency)
    if (count < cap) {
      if (lane == 0) win[(head + count) % cap] = L;
      __syncwarp();
      srt.insert_at(srt.count_less(L), L);
      count += 1;
    } else {
      const double old = win[head];
      __syncwarp();
      if (lane == 0) win[head] = L;
      head = (head + 1) % cap;
      const int at = srt.find(old, count);
      if (at >= 0) srt.remove_at(at);  // (not found only for NaN latencies)
      srt.insert_at(srt.count_less(L), L);
    }
    const int rank = (int)ceil(f64_mul(0.95, (double)count));  // ceil(95.0/100.0 * n)
    p95 = srt.at(rank - 1);
    ch_observe(ce, ewma);
    ch_observe(cq, (double)Q);
    ch_observe(cp, p95);
    outc += 1;
    if (set_qd) last_qd = Q;
  }
  }
  }
  __syncwarp();
  if (slots && fifo && lane == 0) {  // global queue depth seen by this rank's next snapshot
    int64_t extra = 0;
    for (int gi = 0; gi < G; ++gi)
      if (gi != rank) extra += (int64_t)slots[(int64_t)gi * (3 * B + 8) + 3 * B + 1];
    fifo->extra_depth = extra;
  }
  if (slots && lane == 0) {
    st->admitted_total += adm_other;
    st->skipped_total += skip_other;
  }
  for (int i = lane; i < cap; i += 32) st->win[i] = win[i];
  srt.store(st->win_sorted, count);
  if (lane == 0) {
    st->ewma_joules_per_request = ewma;
    st->total_joules = total;
    st->samples_seen = seen;
    st->p95_current = p95;
    st->n_energy = ce;
    st->n_queue_depth = cq;
    st->n_p95_ms = cp;
    st->win_count = count;
    st->win_head = head;
    st->outcomes_total = outc;
    st->queue_depth = last_qd;
    if (err) *err = bad;
  }
}

template <int S>
__global__ void __launch_bounds__(32) outcome_kernel(gg_params p, gg_state* st, const double* lat,
                                                     const double* jou, const int32_t* qd, int64_t n,
                                                     int set_qd, int64_t* err, const double* slots,
                                                     int G, int B, int rank, gg_fifo* fifo) {
  griddep_wait();   // PDL: the predecessor has completed and flushed
  griddep_launch();
  outcome_seq<S>(p, st, lat, jou, qd, n, set_qd, err, slots, G, B, rank, fifo);
}

// ---------------------------------------------------------------------------
// K2, parallel form (same results): the EWMA / totals / channel observes are a
// cheap sequential chain (one thread, CPython order), but the p95 after each
// outcome — the expensive part of the sequential kernel — depends only on the
// latency sequence: outcome i's window is the last min(W, h + i + 1) latencies
// of (history ++ batch), so one warp per outcome selects its nearest-rank
// element (telemetry.py:35-46) independently: the (count - k + 1)-th largest,
// extracted by repeated warp max (ties counted with multiplicity).  The ring
// buffer and the sorted window are rebuilt at the end (positions as the
// deque's appends would leave them).  NaN latencies (whose sorted() order the
// sequential kernel models) fall back to outcome_seq.
constexpr int kOutThreads = 512;   // the largest windows (S >= 16); smaller ones run 1024
template <int S>
struct OutCfg {
  // p95 selection is one warp per outcome: more warps, more outcomes at once
  // (registers: v[S] / kv[S] per lane, so the widest windows keep 512 threads)
  static constexpr int kThreads = S <= 8 ? 1024 : 512;
};
constexpr int kOutChunk = 512;
constexpr int kOutMaxSlots = 64;

// Order-preserving uint64 key of a non-NaN double (NaNs take the sequential
// kernel), with -0.0 mapped onto +0.0 so the zeros compare equal as in Python;
// key 0 is below every real value (the "removed" sentinel).
__device__ __forceinline__ unsigned long long order_ukey(double x) {
  long long b = __double_as_longlong(x);
  if ((b << 1) == 0) b = 0;
  return b < 0 ? (unsigned long long)(~b) : ((unsigned long long)b | 0x8000000000000000ULL);
}

// Nearest-rank p95 (telemetry.py:35-46) of seq[start, start + cnt) for one warp:
// the (cnt - k + 1)-th largest, k = ceil(0.95 cnt), extracted in CPython's
// stable-sort order (equal values -- e.g. -0.0 / +0.0 -- latest arrival first).
template <int S>
__device__ __forceinline__ double p95_select(const double* seq, int start, int cnt, int lane) {
  double v[S];
  unsigned long long kv[S];
#pragma unroll
  for (int q = 0; q < S; ++q) {
    const int j = q * 32 + lane;
    v[q] = j < cnt ? seq[start + j] : 0.0;
    kv[q] = j < cnt ? order_ukey(v[q]) : 0ULL;
  }
  const int k = (int)ceil(f64_mul(0.95, (double)cnt));   // ceil(95.0/100.0 * n)
  const int r = cnt - k + 1;                             // k-th smallest = r-th largest
  double got = 0.0;
  if constexpr (S <= 8) {
    // Same extraction order, cheaper rounds: each lane sorts its S (key,
    // position) pairs once (key descending, later position first), so a
    // round only reduces the lanes' heads and the winning lane shifts its
    // list (the general loop below re-scans all S keys every round).
    unsigned ps[S];
#pragma unroll
    for (int q = 0; q < S; ++q) ps[q] = (unsigned)(q * 32 + lane + 1);
#pragma unroll
    for (int x = 0; x < S; ++x)
#pragma unroll
      for (int y = S - 1; y > x; --y) {
        const bool sw = kv[y] > kv[y - 1] || (kv[y] == kv[y - 1] && ps[y] > ps[y - 1]);
        if (sw) {
          const unsigned long long tk = kv[y];
          kv[y] = kv[y - 1];
          kv[y - 1] = tk;
          const double tv = v[y];
          v[y] = v[y - 1];
          v[y - 1] = tv;
          const unsigned tp = ps[y];
          ps[y] = ps[y - 1];
          ps[y - 1] = tp;
        }
      }
    #pragma unroll 1
    for (int it = 0; it < r; ++it) {
      const unsigned hi = (unsigned)(kv[0] >> 32), lo = (unsigned)kv[0];
      const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
      const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
      const bool cand = hi == mh && lo == ml;
      const unsigned pos = __reduce_max_sync(0xffffffffu, cand ? ps[0] : 0u);
      const int wl = (int)((pos - 1u) & 31u);
      got = __shfl_sync(0xffffffffu, v[0], wl);
      if (lane == wl) {
#pragma unroll
        for (int q = 0; q + 1 < S; ++q) {
          kv[q] = kv[q + 1];
          v[q] = v[q + 1];
          ps[q] = ps[q + 1];
        }
        kv[S - 1] = 0ULL;
        ps[S - 1] = 0u;
      }
    }
  } else {
  #pragma unroll 1
  for (int it = 0; it < r; ++it) {
    unsigned long long bk = kv[0];
    int bq = 0;
#pragma unroll
    for (int q = 1; q < S; ++q)
      if (kv[q] >= bk) {   // ties: the later position (q * 32 + lane grows with q)
        bk = kv[q];
        bq = q;
      }
    const unsigned hi = (unsigned)(bk >> 32), lo = (unsigned)bk;
    const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
    const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
    const bool cand = hi == mh && lo == ml;
    const unsigned pos = __reduce_max_sync(0xffffffffu, cand ? (unsigned)(bq * 32 + lane + 1) : 0u) - 1u;
    const int wl = (int)(pos & 31u), wq = (int)(pos >> 5);
    double wv = 0.0;
#pragma unroll
    for (int q = 0; q < S; ++q)
      if (q == wq) wv = v[q];
    got = __shfl_sync(0xffffffffu, wv, wl);
    if (lane == wl) {
#pragma unroll
      for (int q = 0; q < S; ++q)
        if (q == wq) kv[q] = 0ULL;
    }
  }
  }
  return got;
}

// The p95 after every outcome is independent across outcomes: spread over CTAs
// (kP95PerCta outcomes each, one warp per outcome) ahead of the one-CTA chain
// kernel, which then reads them (outcome_par_kernel's p95_pre).  The window of
// outcome e is the last min(W, h0 + e + 1) latencies of (history ++ batch).
constexpr int kP95PerCta = 64;
constexpr int kP95Threads = 256;
template <int S>
__global__ void __launch_bounds__(kP95Threads) outcome_p95_kernel(gg_params p, const gg_state* st,
                                                                  const double* lat, int64_t n,
                                                                  const double* slots, int G, int B,
                                                                  double* out) {
  griddep_wait();   // PDL: the predecessor has completed and flushed
  griddep_launch();
  __shared__ double seq[GG_P95_WINDOW_MAX + kP95PerCta];
  __shared__ int64_t slot_off[kOutMaxSlots + 1];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cap = p.p95_window;
  const int count0 = st->win_count, head0 = st->win_head;
  if (tid == 0 && slots) {
    int64_t off = 0;
    #pragma unroll 1
    for (int gi = 0; gi < G; ++gi) {
      slot_off[gi] = off;
      off += (int64_t)slots[(int64_t)gi * (3 * B + 8) + 3 * B];
    }
    slot_off[G] = off;
  }
  __syncthreads();
  const int64_t n_tot = slots ? slot_off[G] : n;
  const int64_t e_lo = (int64_t)blockIdx.x * kP95PerCta;
  if (e_lo >= n_tot) return;
  const int64_t e_hi = min(n_tot, e_lo + kP95PerCta);
  const int64_t lo_pos = max((int64_t)0, (int64_t)count0 + e_lo + 1 - cap), hi_pos = count0 + e_hi;
  #pragma unroll 1
  for (int64_t j = tid; j < hi_pos - lo_pos; j += kP95Threads) {
    const int64_t pos = lo_pos + j;
    double L;
    if (pos < count0) {
      L = st->win[(head0 + pos) % cap];
    } else if (slots) {
      const int64_t e = pos - count0;
      int gi = 0;
      while (e >= slot_off[gi + 1]) ++gi;
      L = slots[(int64_t)gi * (3 * B + 8) + (e - slot_off[gi])];
    } else {
      L = lat[pos - count0];
    }
    seq[j] = L;
  }
  __syncthreads();
  #pragma unroll 1
  for (int64_t e = e_lo + warp; e < e_hi; e += kP95Threads / 32) {
    const int cnt = (int)min((int64_t)cap, count0 + e + 1);
    const int start = (int)(count0 + e + 1 - cnt - lo_pos);
    const double got = p95_select<S>(seq, start, cnt, lane);
    if (lane == 0) out[e] = got;
  }
}

template <int S>
__global__ void __launch_bounds__(OutCfg<S>::kThreads) outcome_par_kernel(
    gg_params p, gg_state* st, const double* lat, const double* jou, const int32_t* qd, int64_t n,
    int set_qd, int64_t* err, const double* slots, int G, int B, int rank, gg_fifo* fifo,
    const double* p95_pre) {
  constexpr int kOutThreadsS = OutCfg<S>::kThreads;
  griddep_wait();   // PDL: the predecessor has completed and flushed
  griddep_launch();
  __shared__ double seq[GG_P95_WINDOW_MAX + kOutChunk];   // window history ++ chunk latencies
  __shared__ double sj[kOutChunk];
  __shared__ int32_t sq[kOutChunk];
  __shared__ double sp[kOutChunk];
  __shared__ double sew[kOutChunk];   // EWMA after each outcome (energy channel observes)
  __shared__ double s_ewma, s_total;  // the EWMA chain's results (last warp -> thread 0)
  __shared__ int64_t s_seen;
  __shared__ int64_t slot_off[kOutMaxSlots + 1];
  __shared__ int s_flag, s_first;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cap = p.p95_window;
  const int count0 = st->win_count, head0 = st->win_head;
  // total outcome count and the slot prefix (slots mode)
  if (tid == 0) {
    s_flag = 0;
    int64_t off = 0;
    if (slots) {
      #pragma unroll 1
      for (int gi = 0; gi < G; ++gi) {
        slot_off[gi] = off;
        off += (int64_t)slots[(int64_t)gi * (3 * B + 8) + 3 * B];
      }
      slot_off[G] = off;
    }
  }
  #pragma unroll 1
  for (int j = tid; j < count0; j += kOutThreadsS) seq[j] = st->win[(head0 + j) % cap];
  __syncthreads();
  const int64_t n_tot = slots ? slot_off[G] : n;
  // NaN latencies anywhere -> the sequential kernel's semantics
  bool nan_here = false;
  #pragma unroll 1
  for (int j = tid; j < count0; j += kOutThreadsS) nan_here |= isnan(seq[j]);
  // one pass over the outcomes: NaN check, and the first chunk's (latency, joules,
  // depth) staged in smem for the chunk loop (one global round trip instead of two)
  #pragma unroll 1
  for (int64_t e = tid; e < n_tot; e += kOutThreadsS) {
    double L, J;
    int32_t Q;
    if (slots) {
      int gi = 0;
      while (e >= slot_off[gi + 1]) ++gi;
      const double* sl = slots + (int64_t)gi * (3 * B + 8);
      const int64_t i = e - slot_off[gi];
      L = sl[i];
      J = sl[B + i];
      Q = (int32_t)sl[2 * B + i];
    } else {
      L = lat[e];
      J = jou[e];
      Q = qd[e];
    }
    // a NaN joule makes the EWMA NaN, whose min/max observes are order-dependent in a
    // way the parallel ordered reduction below does not model: sequential kernel
    nan_here |= isnan(L) || isnan(J);
    if (e < kOutChunk) {
      seq[count0 + e] = L;
      sj[e] = J;
      sq[e] = Q;
    }
  }
  if (__syncthreads_or(nan_here)) {
    if (warp == 0) outcome_seq<S>(p, st, lat, jou, qd, n, set_qd, err, slots, G, B, rank, fifo);
    return;
  }
  // thread 0's sequential state (CPython order)
  double ewma = st->ewma_joules_per_request, total = st->total_joules, p95 = st->p95_current;
  int64_t seen = st->samples_seen, outc = st->outcomes_total;
  gg_channel ce = st->n_energy, cq = st->n_queue_depth, cp = st->n_p95_ms;
  int last_qd = st->queue_depth;
  const double lam = p.ewma_lambda, one_minus_lam = f64_sub(1.0, p.ewma_lambda);
  int64_t adm_other = 0, skip_other = 0;
  if (slots && tid == 0) {   // other ranks' admission effects first (see outcome_seq)
    #pragma unroll 1
    for (int gi = 0; gi < G; ++gi) {
      if (gi == rank) continue;
      const double* sl = slots + (int64_t)gi * (3 * B + 8) + 3 * B;
      if (sl[2] - sl[3] > 0.0) {
        if (seen > 0) ch_observe(ce, ewma);
        ch_observe(cq, sl[6]);
        ch_observe(cp, sl[7]);
      }
      adm_other += (int64_t)sl[4];
      skip_other += (int64_t)sl[5];
    }
  }
  int h = count0;            // history length held in seq[0, h)
  int64_t bad = -1, m_total = 0;
  #pragma unroll 1
  for (int64_t e0 = 0; e0 < n_tot && bad < 0; e0 += kOutChunk) {
    const int cn = (int)min((int64_t)kOutChunk, n_tot - e0);
    if (tid == 0) s_first = cn;
    __syncthreads();
    #pragma unroll 1
    for (int c = tid; c < cn; c += kOutThreadsS) {
      const int64_t e = e0 + c;
      double L, J;
      int32_t Q;
      if (e0 == 0) {   // staged by the NaN pass (h == count0 here)
        L = seq[h + c];
        J = sj[c];
        Q = sq[c];
      } else if (slots) {
        int gi = 0;
        while (e >= slot_off[gi + 1]) ++gi;
        const double* sl = slots + (int64_t)gi * (3 * B + 8);
        const int64_t i = e - slot_off[gi];
        L = sl[i];
        J = sl[B + i];
        Q = (int32_t)sl[2 * B + i];
      } else {
        L = lat[e];
        J = jou[e];
        Q = qd[e];
      }
      seq[h + c] = L;
      sj[c] = J;
      sq[c] = Q;
      if (L < 0.0 || J < 0.0 || Q < 0) atomicMin(&s_first, c);   // NegativeMeasurement
    }
    __syncthreads();
    const int nc = s_first;
    if (nc < cn) {
      const int64_t e = e0 + nc;
      if (slots) {
        int gi = 0;
        while (e >= slot_off[gi + 1]) ++gi;
        bad = (int64_t)gi * B + (e - slot_off[gi]);
      } else {
        bad = e;
      }
    }
    // the order-dependent chains, one thread in CPython order — the EWMA recurrence
    // (energy.py:24-36, 75-87) and the running total — on the last warp, which
    // takes no p95 work, so the chain overlaps the p95 selection below.  The
    // products (1 - lam) * J are order-independent: the warp forms them first
    // (into sew), and the chain e = fl(fl(lam e) + t) runs on registers, eight
    // outcomes' terms loaded ahead of their step.
    if (warp == kOutThreadsS / 32 - 1) {
      #pragma unroll 1
      for (int c = lane; c < nc; c += 32) sew[c] = f64_mul(one_minus_lam, sj[c]);
      __syncwarp();
      if (lane == 0) {
        const int64_t seen0 = seen;
        int c = 0;
        if (seen == 0 && nc > 0) {   // the first sample seeds the average
          ewma = sj[0];
          total = f64_add(total, sj[0]);
          sew[0] = ewma;
          seen = 1;
          c = 1;
        }
        #pragma unroll 1
        for (; c + 8 <= nc; c += 8) {
          double t[8], jv[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            t[q] = sew[c + q];
            jv[q] = sj[c + q];
          }
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            ewma = f64_add(f64_mul(lam, ewma), t[q]);
            total = f64_add(total, jv[q]);
            t[q] = ewma;
          }
#pragma unroll
          for (int q = 0; q < 8; ++q) sew[c + q] = t[q];
        }
        #pragma unroll 1
        for (; c < nc; ++c) {
          ewma = f64_add(f64_mul(lam, ewma), sew[c]);
          total = f64_add(total, sj[c]);
          sew[c] = ewma;
        }
        seen = seen0 + nc;
        s_ewma = ewma;
        s_total = total;
        s_seen = seen;
      }
    }
    // p95 after each outcome: precomputed by outcome_p95_kernel, or here with one
    // warp per outcome (all warps but the chain's)
    if (p95_pre) {
      #pragma unroll 1
      for (int c = tid; c < nc; c += kOutThreadsS) sp[c] = p95_pre[e0 + c];
    }
    #pragma unroll 1
    for (int c = warp; !p95_pre && c < nc && warp < kOutThreadsS / 32 - 1; c += kOutThreadsS / 32 - 1) {
      const int cnt = min(cap, h + c + 1);
      const int start = h + c + 1 - cnt;
      const double got = p95_select<S>(seq, start, cnt, lane);
      if (lane == 0) sp[c] = got;
    }
    __syncthreads();
    if (tid == 0) {
      ewma = s_ewma;
      total = s_total;
      seen = s_seen;
      outc += nc;
      if (nc > 0) {
        p95 = sp[nc - 1];
        if (set_qd) last_qd = sq[nc - 1];
      }
    }
    __syncthreads();
    // NormalizerChannel.observe (controller.py:164-168) over each outcome's energy /
    // queue-depth / p95 value: a fold with "replace only if strictly smaller /
    // larger", associative without NaNs (guaranteed above) and order-preserving on
    // ties, so warp 0 folds contiguous segments per lane and combines them in lane
    // order; lane 0 (thread 0) folds the running channels in first.
    if (warp == 0 && nc > 0) {
      const int seg = (nc + 31) / 32;
      const int c0 = min(nc, lane * seg), c1 = min(nc, c0 + seg);
      double lo[3], hi[3];
      bool has = c0 < c1;
      if (has) {
        lo[0] = hi[0] = sew[c0];
        lo[1] = hi[1] = (double)sq[c0];
        lo[2] = hi[2] = sp[c0];
        #pragma unroll 1
        for (int c = c0 + 1; c < c1; ++c) {
          const double x0 = sew[c], x1 = (double)sq[c], x2 = sp[c];
          if (x0 < lo[0]) lo[0] = x0;
          if (x0 > hi[0]) hi[0] = x0;
          if (x1 < lo[1]) lo[1] = x1;
          if (x1 > hi[1]) hi[1] = x1;
          if (x2 < lo[2]) lo[2] = x2;
          if (x2 > hi[2]) hi[2] = x2;
        }
      } else {
#pragma unroll
        for (int k = 0; k < 3; ++k) lo[k] = hi[k] = 0.0;
      }
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {   // combine (this, lane + o) as (left, right)
        const bool rhas = __shfl_down_sync(0xffffffffu, (int)has, o) != 0;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const double rlo = __shfl_down_sync(0xffffffffu, lo[k], o);
          const double rhi = __shfl_down_sync(0xffffffffu, hi[k], o);
          if ((lane & (2 * o - 1)) == 0 && lane + o < 32 && rhas) {
            if (!has || rlo < lo[k]) lo[k] = rlo;
            if (!has || rhi > hi[k]) hi[k] = rhi;
          }
        }
        if ((lane & (2 * o - 1)) == 0 && lane + o < 32) has = has || rhas;
      }
      if (lane == 0 && has) {
        gg_channel* ch[3] = {&ce, &cq, &cp};
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          gg_channel& c = *ch[k];
          if (!c.seen || lo[k] < c.lo) c.lo = lo[k];
          if (!c.seen || hi[k] > c.hi) c.hi = hi[k];
          c.seen = 1;
        }
      }
    }
    // keep the last min(cap, h + nc) latencies as the next history
    const int hn = min(cap, h + nc), src = h + nc - hn;
    double tmp[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int j = tid + q * kOutThreadsS;
      tmp[q] = j < hn ? seq[src + j] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int j = tid + q * kOutThreadsS;
      if (j < hn) seq[j] = tmp[q];
    }
    h = hn;
    m_total += nc;
    __syncthreads();
  }
  // ring buffer: window element j sits at (head_f + j) % cap
  const int head_f = (count0 + m_total <= cap) ? head0 : (int)((head0 + (count0 + m_total - cap)) % cap);
  #pragma unroll 1
  for (int j = tid; j < h; j += kOutThreadsS) st->win[(head_f + j) % cap] = seq[j];
  // sorted window = CPython's stable sorted(): each element lands at its stable rank
  // (smaller values, then equal values earlier in arrival order): h^2 / 512 compares
  // against the smem window instead of a bitonic network's syncs
  #pragma unroll 1
  for (int j = tid; j < h; j += kOutThreadsS) {
    const double vj = seq[j];
    int rk = 0;
    #pragma unroll 4
    for (int i = 0; i < h; ++i) {
      const double vi = seq[i];
      rk += (vi < vj || (vi == vj && i < j)) ? 1 : 0;
    }
    st->win_sorted[rk] = vj;
  }
  if (tid == 0) {
    if (slots && fifo) {   // global queue depth seen by this rank's next snapshot
      int64_t extra = 0;
      #pragma unroll 1
      for (int gi = 0; gi < G; ++gi)
        if (gi != rank) extra += (int64_t)slots[(int64_t)gi * (3 * B + 8) + 3 * B + 1];
      fifo->extra_depth = extra;
    }
    if (slots) {
      st->admitted_total += adm_other;
      st->skipped_total += skip_other;
    }
    st->ewma_joules_per_request = ewma;
    st->total_joules = total;
    st->samples_seen = seen;
    st->p95_current = p95;
    st->n_energy = ce;
    st->n_queue_depth = cq;
    st->n_p95_ms = cp;
    st->win_count = h;
    st->win_head = head_f;
    st->outcomes_total = outc;
    st->queue_depth = last_qd;
    if (err) *err = bad;
  }
}

__global__ void state_scalar_kernel(gg_state* st, int which, double t, int32_t q) {
  if (threadIdx.x != 0) return;
  if (which == 0) st->t_origin = t;
  else st->queue_depth = q;
}

// ---------------------------------------------------------------------------
// K3: fp32 logits -> fp64 probabilities, one warp per row.  Probabilities are
// exp((double)x - max) / sum in fp64, so |sum(p) - 1| is a few ulp and the rows
// pass _validate_distribution (controller.py:132-134); fp32 rows would not.
__global__ void __launch_bounds__(256) epilogue_kernel(const float* logits, int64_t n, int32_t k,
                                                       int64_t ld, int32_t proxy, double ln_k,
                                                       double* probs, int32_t* argmax,
                                                       double* conf, double* util) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (row >= n) return;
  const float* x = logits + row * ld;
  float m = -INFINITY;
  for (int j = lane; j < k; j += 32) m = fmaxf(m, x[j]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  const double md = (double)m;
  double s = 0.0;
  for (int j = lane; j < k; j += 32) s += exp((double)x[j] - md);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const double inv = 1.0 / s;
  double best = -1.0;
  int bi = 0x7fffffff;
  double* prow = probs ? probs + row * (int64_t)k : nullptr;
  for (int j = lane; j < k; j += 32) {
    double pj = exp((double)x[j] - md) * inv;
    if (prow) prow[j] = pj;
    if (pj > best) {
      best = pj;
      bi = j;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double ob = __shfl_xor_sync(0xffffffffu, best, o);
    int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ob > best || (ob == best && oi < bi)) {
      best = ob;
      bi = oi;
    }
  }
  if (lane == 0) {
    if (argmax) argmax[row] = bi;
    if (conf) conf[row] = best;
  }
  if (util && prow) {
    __syncwarp();
    if (lane == 0) {  // the controller's own sequential utility of the written row
      RowAcc acc;
      const bool entropy = proxy == GG_UTIL_ENTROPY;
      for (int j = 0; j < k; ++j) acc.add(prow[j], entropy);
      double u;
      util[row] = acc.finish(k, entropy, ln_k, u) ? u : __longlong_as_double(0x7ff8000000000000ll);
    }
  }
}

// Stateless batch forms (gg_utility / gg_threshold / gg_cost).
__global__ void utility_kernel(const double* probs, int64_t n, int32_t k, int64_t stride,
                               int32_t proxy, double ln_k, double* util, uint8_t* valid) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const bool entropy = proxy == GG_UTIL_ENTROPY;
  RowAcc acc;
  for (int c = 0; c < k; ++c) acc.add(probs[r * stride + c], entropy);
  double u;
  const bool ok = acc.finish(k, entropy, ln_k, u);
  if (util) util[r] = ok ? u : __longlong_as_double(0x7ff8000000000000ll);
  if (valid) valid[r] = ok ? 1 : 0;
}

__global__ void threshold_kernel(double tau0, double tau_inf, double k, double t_origin,
                                 const double* t, double* tau, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double el = f64_sub(t[i], t_origin);
  el = (el > 0.0) ? el : 0.0;
  tau[i] = f64_add(tau_inf, f64_mul(f64_sub(tau0, tau_inf), exp(f64_mul(-k, el))));
}

__global__ void cost_kernel(double alpha, double beta, double gamma, const double* uec, double* j,
                            int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  j[i] = f64_add(f64_add(f64_mul(alpha, uec[3 * i]), f64_mul(beta, uec[3 * i + 1])),
                 f64_mul(gamma, uec[3 * i + 2]));
}

}  // namespace gg

// ===========================================================================
// C ABI
using namespace gg;

extern "C" {

const char* gg_version(void) { return "greengate-b200 0.1.0 (sm_100a)"; }
int gg_abi_version(void) { return GG_ABI_VERSION; }
size_t gg_state_bytes(void) { return sizeof(gg_state); }

int gg_validate_params(const gg_params* p) {
  if (!p) return GG_ERR_INVALID_ARGUMENT;
  // CostWeights.__post_init__ (controller.py:85-88) -> ValueError
  if (!(isfinite(p->alpha) && isfinite(p->beta) && isfinite(p->gamma))) return GG_ERR_INVALID_ARGUMENT;
  // ThresholdSchedule.__post_init__ (controller.py:100-105)
  if (!(isfinite(p->tau0) && isfinite(p->tau_inf) && isfinite(p->k))) return GG_ERR_INVALID_SCHEDULE;
  if (p->k <= 0.0) return GG_ERR_INVALID_SCHEDULE;
  // EnergyLedger.__post_init__ (energy.py:64-69)
  if (!(isfinite(p->ewma_lambda) && p->ewma_lambda > 0.0 && p->ewma_lambda < 1.0)) return GG_ERR_INVALID_LAMBDA;
  if (p->direction < 0 || p->direction > 1) return GG_ERR_INVALID_ARGUMENT;
  if (p->utility_proxy < 0 || p->utility_proxy > 1) return GG_ERR_INVALID_ARGUMENT;
  if (p->routing < 0 || p->routing > 2) return GG_ERR_INVALID_ARGUMENT;
  if (p->p95_window < 1 || p->p95_window > GG_P95_WINDOW_MAX) return GG_ERR_INVALID_ARGUMENT;
  return GG_OK;
}

int gg_state_init(gg_state* state_dev, double t_origin, void* stream) {
  if (!state_dev) return GG_ERR_INVALID_ARGUMENT;
  if (!isfinite(t_origin)) return GG_ERR_INVALID_SCHEDULE;
  cudaStream_t s = gg_stream(stream);
  GG_CUDA_OK(cudaMemsetAsync(state_dev, 0, sizeof(gg_state), s));
  state_scalar_kernel<<<1, 32, 0, s>>>(state_dev, 0, t_origin, 0);
  GG_LAUNCH_OK();
  return GG_OK;
}

int gg_reset_clock(gg_state* state_dev, double t_origin, void* stream) {
  if (!state_dev) return GG_ERR_INVALID_ARGUMENT;
  if (!isfinite(t_origin)) return GG_ERR_INVALID_SCHEDULE;
  state_scalar_kernel<<<1, 32, 0, gg_stream(stream)>>>(state_dev, 0, t_origin, 0);
  GG_LAUNCH_OK();
  return GG_OK;
}

int gg_set_queue_depth(gg_state* state_dev, int32_t queue_depth, void* stream) {
  if (!state_dev || queue_depth < 0) return GG_ERR_INVALID_ARGUMENT;
  state_scalar_kernel<<<1, 32, 0, gg_stream(stream)>>>(state_dev, 1, 0.0, queue_depth);
  GG_LAUNCH_OK();
  return GG_OK;
}

static int num_sms_cached() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) sms = 148;
  }
  return sms;
}

static int64_t admit_blocks(int64_t n, int32_t k) {
  const int64_t rows_per_block = (k <= 16) ? kSmallThreads * kSmallRpt : kLargeRows;
  int64_t nb = (n + rows_per_block - 1) / rows_per_block;
  return nb < 1 ? 1 : nb;
}

static int64_t lookback_words(int64_t n) {   // worst case over the single-pass kernels
  const int64_t nb = (n + kFastRows - 1) / kFastRows;
  return nb < 1 ? 1 : nb;
}

size_t gg_admit_workspace_bytes(int64_t n) {
  // look-back words + split-path counters (decide-block counts + super sums)
  const int64_t nbs = (n + kDecideRows - 1) / kDecideRows + 1;
  return kWsHeader + sizeof(unsigned long long) * (size_t)(lookback_words(n) + 2 * nbs);
}

static int launch_admit(const AdmitArgs& a, void* stream);

// K2 instantiation by window capacity (register slots per lane = ceil(W / 32)).
// Per-controller scratch for the p95 pre-pass (one double per outcome), keyed by
// the state's device address; grown outside stream capture only (inside a
// capture without room, the chain kernel computes the p95s itself).
static std::mutex g_p95_mu;
static std::unordered_map<const gg_state*, std::pair<double*, int64_t>> g_p95_scratch;
static double* p95_scratch(const gg_state* st, int64_t need, cudaStream_t s) {
  std::lock_guard<std::mutex> lk(g_p95_mu);
  auto& e = g_p95_scratch[st];
  if (e.second >= need) return e.first;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return nullptr;
  const int64_t cap = need < 4096 ? 4096 : need;
  double* ptr = nullptr;
  if (cudaMalloc(&ptr, cap * sizeof(double)) != cudaSuccess) return nullptr;
  if (e.first) {
    cudaStreamSynchronize(s);   // the old scratch may still be read by queued work
    cudaFree(e.first);
  }
  e = {ptr, cap};
  return ptr;
}

static int launch_outcome(const gg_params& p, gg_state* st, const double* lat, const double* jou,
                          const int32_t* qd, int64_t n, int set_qd, int64_t* err,
                          const double* slots, int G, int B, int rank, gg_fifo* fifo,
                          void* stream) {
  cudaStream_t s = gg_stream(stream);
  const int w = p.p95_window;
  const bool par = !getenv("GG_OUTCOME_SEQ") && (!slots || G <= kOutMaxSlots);
  // p95 pre-pass over several CTAs once there are enough outcomes to spread
  static const bool no_pre = getenv("GG_OUTCOME_NO_PRE") != nullptr;
  const int64_t n_max = slots ? (int64_t)G * B : n;
  // (>= 64 outcomes: one serving batch's p95s in parallel; the chain kernel's
  // sequential p95 made K2 ~20 us at B = 128, on the pipelined step's critical tail)
  static const int pre_min = getenv("GG_OUTCOME_PRE_MIN") ? atoi(getenv("GG_OUTCOME_PRE_MIN")) : kP95PerCta;
  double* pre = (par && !no_pre && n_max >= pre_min) ? p95_scratch(st, n_max, s) : nullptr;
  const unsigned pre_grid = (unsigned)((n_max + kP95PerCta - 1) / kP95PerCta);
#define GG_OUTCOME(SLOTS)                                                                        \
  do {                                                                                           \
    if (par && pre)                                                                              \
      GG_PDL_LAUNCH((outcome_p95_kernel<SLOTS>), pre_grid, kP95Threads, 0, s, p, st, lat, n, slots, G, B, pre); \
    if (par)                                                                                     \
      GG_PDL_LAUNCH((outcome_par_kernel<SLOTS>), 1, OutCfg<SLOTS>::kThreads, 0, s, p, st, lat, jou, qd, n, set_qd, err, slots, \
                                                          G, B, rank, fifo, (const double*)pre); \
    else                                                                                         \
      GG_PDL_LAUNCH((outcome_kernel<SLOTS>), 1, 32, 0, s, p, st, lat, jou, qd, n, set_qd, err, slots, G, B,   \
                                             rank, fifo);                                        \
  } while (0)
  if (w <= 32) GG_OUTCOME(1);
  else if (w <= 64) GG_OUTCOME(2);
  else if (w <= 128) GG_OUTCOME(4);
  else if (w <= 256) GG_OUTCOME(8);
  else if (w <= 512) GG_OUTCOME(16);
  else GG_OUTCOME(32);
#undef GG_OUTCOME
  GG_LAUNCH_OK();
  return GG_OK;
}

int gg_admit(const gg_params* params, gg_state* state_dev, const double* probs_dev, int64_t n,
             int32_t k, int64_t row_stride, const double* now_dev, const gg_snapshot* snapshot_dev,
             uint8_t* decision_dev, double* breakdown_dev, int32_t* admitted_idx_dev,
             gg_batch_info* info_dev, void* workspace_dev, size_t workspace_bytes, void* stream) {
  int rc = gg_validate_params(params);
  if (rc != GG_OK) return rc;
  if (!state_dev || !workspace_dev || n < 0 || k < 1 || row_stride < k)
    return GG_ERR_INVALID_ARGUMENT;
  if (n > 0 && (!probs_dev || !now_dev || !decision_dev)) return GG_ERR_INVALID_ARGUMENT;
  if (n > (int64_t)0x7fffffff) return GG_ERR_UNSUPPORTED;  // int32 admitted indices
  if (workspace_bytes < gg_admit_workspace_bytes(n)) return GG_ERR_INVALID_ARGUMENT;
  AdmitArgs a;
  a.p = *params;
  a.state = state_dev;
  a.probs = probs_dev;
  a.n = n;
  a.k = k;
  a.stride = row_stride;
  a.now = now_dev;
  a.snap = snapshot_dev;
  a.decision = decision_dev;
  a.breakdown = breakdown_dev;
  a.admitted_idx = admitted_idx_dev;
  a.info = info_dev;
  a.ws = reinterpret_cast<AdmitWorkspace*>(workspace_dev);
  a.ln_k = log((double)k);  // host libm == CPython math.log (controller.py:142)
  a.fifo = nullptr;
  a.ring = nullptr;
  a.ring_ns = nullptr;
  return launch_admit(a, stream);
}

static int launch_admit(const AdmitArgs& args, void* stream) {
  AdmitArgs a = args;
  const int64_t n = a.n;
  const int32_t k = a.k;
  const int64_t nb = admit_blocks(n, k);
  cudaStream_t s = gg_stream(stream);
  const bool aligned16 = ((reinterpret_cast<uintptr_t>(a.probs) & 15) == 0) && (a.stride % 2 == 0);
  const bool bd = a.breakdown != nullptr;
  if (k <= 16) {
    // large batches: decide / scan / compact (three launches, no cross-block
    // waiting); the serving window (FIFO mode, small n): single pass with a
    // decoupled look-back
    static const int split_env = getenv("GG_K1_SPLIT") ? atoi(getenv("GG_K1_SPLIT")) : -1;
    const bool split = split_env >= 0 ? (split_env != 0 && !a.fifo)
                                      : (!a.fifo && nb >= 4 * num_sms_cached());
    const unsigned g = (unsigned)nb;
    if (split) {   // counters after the look-back words (gg_admit_workspace_bytes)
      int sh = 2;
      while ((1ll << (2 * sh)) < nb) ++sh;   // 2^sh >= sqrt(nb)
      a.super_shift = sh;
      a.split_cnt = a.ws->status + lookback_words(n);
      a.super_cnt = a.split_cnt + nb;
    }
    if (split) {
      GG_PDL_LAUNCH((admit_prologue_kernel), 1, 32, 0, s, a);
      GG_LAUNCH_OK();
    }
    const bool ent = a.p.utility_proxy == GG_UTIL_ENTROPY;
#define GG_SMALL(KC)                                                                        \
  do {                                                                                      \
    if (bd && split) GG_PDL_LAUNCH((admit_small_kernel<KC, kSmallRpt, true, true>), g, kSmallThreads, 0, s, a);    \
    else if (bd) GG_PDL_LAUNCH((admit_small_kernel<KC, kSmallRpt, true, false>), g, kSmallThreads, 0, s, a);      \
    else if (split && ent) GG_PDL_LAUNCH((admit_small_kernel<KC, kSmallRpt, false, true, 1>), g, kSmallThreads, 0, s, a); \
    else if (split) GG_PDL_LAUNCH((admit_small_kernel<KC, kSmallRpt, false, true, 2>), g, kSmallThreads, 0, s, a);        \
    else if (ent) GG_PDL_LAUNCH((admit_small_kernel<KC, kSmallRpt, false, false, 1>), g, kSmallThreads, 0, s, a);         \
    else GG_PDL_LAUNCH((admit_small_kernel<KC, kSmallRpt, false, false, 2>), g, kSmallThreads, 0, s, a);                  \
  } while (0)
    if (k == 2 && aligned16) GG_SMALL(2);
    else if (k == 4 && aligned16) GG_SMALL(4);
    else GG_SMALL(0);
#undef GG_SMALL
    if (split) {
      GG_LAUNCH_OK();
      GG_PDL_LAUNCH((admit_compact_kernel), (unsigned)((n + kCompactRows - 1) / kCompactRows), kSmallThreads, 0, s, 
          a, (int)nb);
    }
  } else if (!bd && !getenv("GG_ADMIT_EXACT_ONLY")) {
    const unsigned g = (unsigned)((n + kFastRows - 1) / kFastRows > 0 ? (n + kFastRows - 1) / kFastRows : 1);
    if (k <= kRegChunks * 32)
      GG_PDL_LAUNCH((admit_large_fast_kernel<true>), g, kFastThreads, 0, s, a);
    else
      GG_PDL_LAUNCH((admit_large_fast_kernel<false>), g, kFastThreads, 0, s, a);
  } else {
    GG_PDL_LAUNCH((admit_large_kernel), (unsigned)nb, kLargeThreads, 0, s, a);
  }
  GG_LAUNCH_OK();
  return GG_OK;
}

int gg_outcome(const gg_params* params, gg_state* state_dev, const double* latency_ms_dev,
               const double* joules_dev, const int32_t* queue_depth_dev, int64_t n,
               int32_t set_queue_depth, int64_t* error_index_dev, void* stream) {
  int rc = gg_validate_params(params);
  if (rc != GG_OK) return rc;
  if (!state_dev || n < 0) return GG_ERR_INVALID_ARGUMENT;
  if (n > 0 && (!latency_ms_dev || !joules_dev || !queue_depth_dev)) return GG_ERR_INVALID_ARGUMENT;
  return launch_outcome(*params, state_dev, latency_ms_dev, joules_dev, queue_depth_dev, n,
                        set_queue_depth, error_index_dev, nullptr, 0, 0, 0, nullptr, stream);
}

int gg_outcome_slots(const gg_params* params, gg_state* state_dev, const double* slots_dev,
                     int32_t G, int32_t B, int32_t rank, gg_fifo* fifo_dev,
                     int64_t* error_index_dev, void* stream) {
  int rc = gg_validate_params(params);
  if (rc != GG_OK) return rc;
  if (!state_dev || !slots_dev || G < 1 || B < 1 || rank < 0 || rank >= G)
    return GG_ERR_INVALID_ARGUMENT;
  return launch_outcome(*params, state_dev, nullptr, nullptr, nullptr, 0, 1, error_index_dev,
                        slots_dev, G, B, rank, fifo_dev, stream);
}

int gg_admit_stream(const gg_params* params, gg_state* state_dev, gg_fifo* fifo_dev,
                    int32_t* ring_ids_dev, uint64_t* ring_ns_dev, const double* probs_dev,
                    int32_t k, int64_t row_stride, const double* now_dev, int64_t window,
                    const gg_snapshot* snapshot_dev, uint8_t* decision_dev,
                    gg_batch_info* info_dev, void* workspace_dev, size_t workspace_bytes,
                    void* stream) {
  int rc = gg_validate_params(params);
  if (rc != GG_OK) return rc;
  if (!state_dev || !fifo_dev || !ring_ids_dev || !probs_dev || !now_dev || !decision_dev ||
      !workspace_dev || window < 1 || k < 1 || row_stride < k)
    return GG_ERR_INVALID_ARGUMENT;
  if (window > (int64_t)0x7fffffff) return GG_ERR_UNSUPPORTED;
  if (workspace_bytes < gg_admit_workspace_bytes(window)) return GG_ERR_INVALID_ARGUMENT;
  AdmitArgs a;
  a.p = *params;
  a.state = state_dev;
  a.probs = probs_dev;
  a.n = window;
  a.k = k;
  a.stride = row_stride;
  a.now = now_dev;
  a.snap = snapshot_dev;
  a.decision = decision_dev;
  a.breakdown = nullptr;
  a.admitted_idx = nullptr;
  a.info = info_dev;
  a.ws = reinterpret_cast<AdmitWorkspace*>(workspace_dev);
  a.ln_k = log((double)k);
  a.fifo = fifo_dev;
  a.ring = ring_ids_dev;
  a.ring_ns = ring_ns_dev;
  return launch_admit(a, stream);
}

int gg_epilogue(const float* logits_dev, int64_t n, int32_t k, int64_t ld, int32_t utility_proxy,
                double* probs_dev, int32_t* argmax_dev, double* confidence_dev, double* utility_dev,
                void* stream) {
  if (!logits_dev || n < 0 || k < 1 || ld < k) return GG_ERR_INVALID_ARGUMENT;
  if (utility_dev && !probs_dev) return GG_ERR_INVALID_ARGUMENT;
  if (n == 0) return GG_OK;
  const int rows_per_block = 8;
  const int64_t nb = (n + rows_per_block - 1) / rows_per_block;
  epilogue_kernel<<<(unsigned)nb, 256, 0, gg_stream(stream)>>>(
      logits_dev, n, k, ld, utility_proxy, log((double)k), probs_dev, argmax_dev, confidence_dev,
      utility_dev);
  GG_LAUNCH_OK();
  return GG_OK;
}

int gg_utility(const double* probs_dev, int64_t n, int32_t k, int64_t row_stride,
               int32_t utility_proxy, double* utility_dev, uint8_t* valid_dev, void* stream) {
  if (n < 0 || k < 1 || row_stride < k || (n > 0 && !probs_dev)) return GG_ERR_INVALID_ARGUMENT;
  if (utility_proxy < 0 || utility_proxy > 1) return GG_ERR_INVALID_ARGUMENT;
  if (n == 0) return GG_OK;
  utility_kernel<<<(unsigned)((n + 127) / 128), 128, 0, gg_stream(stream)>>>(
      probs_dev, n, k, row_stride, utility_proxy, log((double)k), utility_dev, valid_dev);
  GG_LAUNCH_OK();
  return GG_OK;
}

int gg_threshold(double tau0, double tau_inf, double k, double t_origin, const double* t_dev,
                 double* tau_dev, int64_t n, void* stream) {
  // threshold_at re-checks the rate (controller.py:120-121)
  if (!(isfinite(k) && k > 0.0)) return GG_ERR_INVALID_SCHEDULE;
  if (n < 0 || (n > 0 && (!t_dev || !tau_dev))) return GG_ERR_INVALID_ARGUMENT;
  if (n == 0) return GG_OK;
  threshold_kernel<<<(unsigned)((n + 255) / 256), 256, 0, gg_stream(stream)>>>(
      tau0, tau_inf, k, t_origin, t_dev, tau_dev, n);
  GG_LAUNCH_OK();
  return GG_OK;
}

int gg_cost(double alpha, double beta, double gamma, const double* uec_dev, double* j_dev,
            int64_t n, void* stream) {
  if (n < 0 || (n > 0 && (!uec_dev || !j_dev))) return GG_ERR_INVALID_ARGUMENT;
  if (n == 0) return GG_OK;
  cost_kernel<<<(unsigned)((n + 255) / 256), 256, 0, gg_stream(stream)>>>(alpha, beta, gamma,
                                                                          uec_dev, j_dev, n);
  GG_LAUNCH_OK();
  return GG_OK;
}

}  // extern "C"
