// gg_controller.cu — admission (K1), outcome feedback (K2) and logit epilogue
// (K3) kernels of the gated-inference hot path, plus their C-ABI entry points
// (include/greengate_b200.h).
//
// Compiled with -fmad=false; every controller operation additionally goes
// through the __d*_rn intrinsics in gg_common.cuh, so each fp64 binary op
// rounds exactly like CPython's float op in the reference
// (pkg/src/greengate/controller.py, energy.py, telemetry.py).
#include <math.h>
#include <stdio.h>

#include "gg_common.cuh"

namespace gg {

// ---------------------------------------------------------------------------
// Workspace layout (zero-filled once; every gg_admit launch leaves it zeroed).
struct AdmitWorkspace {
  unsigned long long vblock_counter;  // virtual block ids (forward-progress-safe lookback)
  unsigned long long done_counter;    // completion ticket; the last block finalizes
  unsigned long long n_skipped;
  unsigned long long n_invalid;
  unsigned long long first_invalid_enc;  // max over (n - row); 0 == none
  unsigned long long reserved[3];
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

// Single-thread decoupled look-back (Merrill & Garland): returns the exclusive
// prefix of admitted rows before virtual block `vb`.
__device__ unsigned long long lookback(unsigned long long* status, int vb, unsigned long long agg) {
  if (vb == 0) {
    st_relaxed(&status[0], kFlagPrefix | agg);
    return 0ull;
  }
  st_relaxed(&status[vb], kFlagAgg | agg);
  unsigned long long prefix = 0;
  int p = vb - 1;
  while (true) {
    unsigned long long w;
    do {
      w = ld_relaxed(&status[p]);
    } while ((w >> 62) == 0ull);
    prefix += w & kValMask;
    if ((w >> 62) == 2ull) break;
    --p;
  }
  st_relaxed(&status[vb], kFlagPrefix | (prefix + agg));
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
  static constexpr int GROUPS = RPT * WARPS;
  static_assert(GROUPS <= 32, "one warp scans the groups");
  BatchConst bc;
  int64_t row0, nw, depth0;   // window start/length; FIFO depth before this launch
  unsigned long long block_prefix;
  int group_cnt[GROUPS];
  int group_off[GROUPS];
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

// Per-block prologue (thread 0): virtual block id, decision window, FIFO depth
// and the batch-constant E/C — all read before any block can finalize.
template <int THREADS, int RPT>
__device__ void block_setup(const AdmitArgs& a, AdmitShared<THREADS, RPT>& sm) {
  sm.vb = (int)atomicAdd(&a.ws->vblock_counter, 1ull);
  int64_t row0, nw;
  admit_window(a, row0, nw);
  sm.row0 = row0;
  sm.nw = nw;
  sm.depth0 = a.fifo ? a.fifo->tail - a.fifo->head : 0;
  sm.bc = batch_constants(a.state, a.snap, a.fifo);
}

// Order-preserving compaction of the tile + counters + last-block finalize.
template <int THREADS, int RPT>
__device__ void finish_tile(const AdmitArgs& a, AdmitShared<THREADS, RPT>& sm, int64_t tile0,
                            const uint32_t (&ballots)[RPT], int my_skip, int my_inv,
                            unsigned long long my_bad_enc) {
  constexpr int WARPS = THREADS / 32;
  constexpr int GROUPS = RPT * WARPS;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (lane == 0) {
#pragma unroll
    for (int j = 0; j < RPT; ++j) sm.group_cnt[j * WARPS + warp] = __popc(ballots[j]);
  }
  // counters: warp-reduce then one atomic per warp
  int ws = warp_sum(my_skip), wi = warp_sum(my_inv);
  unsigned long long wb = warp_max_u64(my_bad_enc);
  if (lane == 0) {
    if (ws) atomicAdd(&a.ws->n_skipped, (unsigned long long)ws);
    if (wi) atomicAdd(&a.ws->n_invalid, (unsigned long long)wi);
    if (wb) atomicMax(&a.ws->first_invalid_enc, wb);
  }
  __syncthreads();
  if (warp == 0) {
    int c = lane < GROUPS ? sm.group_cnt[lane] : 0;
    int v = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int t = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += t;
    }
    int total = __shfl_sync(0xffffffffu, v, 31);
    if (lane < GROUPS) sm.group_off[lane] = v - c;
    if (lane == 0) sm.block_prefix = lookback(a.ws->status, sm.vb, (unsigned long long)total);
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
    const int nb = gridDim.x;
    unsigned long long w = ld_relaxed(&a.ws->status[nb - 1]);
    int64_t n_adm = (int64_t)(w & kValMask);
    int64_t n_skip = (int64_t)ld_relaxed(&a.ws->n_skipped);
    int64_t n_inv = (int64_t)ld_relaxed(&a.ws->n_invalid);
    unsigned long long benc = ld_relaxed(&a.ws->first_invalid_enc);
    gg_state* st = a.state;
    const BatchConst& b = sm.bc;
    const bool any_valid = (sm.nw - n_inv) > 0;
    if (any_valid) {
      if (b.samples_seen > 0) ch_observe(st->n_energy, b.ewma);
      ch_observe(st->n_queue_depth, (double)b.qd);
      ch_observe(st->n_p95_ms, b.p95);
    }
    st->admitted_total += n_adm;
    st->skipped_total += n_skip;
    if (a.fifo) {
      const int64_t room = a.fifo->capacity - sm.depth0;
      a.fifo->tail += n_adm < room ? n_adm : room;
      a.fifo->cursor = sm.row0 + sm.nw;
    }
    if (a.info) {
      a.info->n_admitted = n_adm;
      a.info->n_skipped = n_skip;
      a.info->n_invalid = n_inv;
      a.info->first_invalid = benc ? (int64_t)(sm.row0 + sm.nw - (int64_t)benc) : -1;
      a.info->energy = any_valid ? b.e : 0.0;
      a.info->congestion = any_valid ? b.c : 0.0;
      a.info->n_decided = sm.nw;
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
  __syncthreads();
  for (int i = tid; i < (int)gridDim.x; i += THREADS) a.ws->status[i] = 0ull;
}

// K1, small K (K <= 16): RPT rows per thread, rows of a warp contiguous, so a
// warp's loads of a [32 x K] fp64 slab are fully coalesced.
template <int KC, int THREADS, int RPT>
__global__ void __launch_bounds__(THREADS) admit_small_kernel(AdmitArgs a) {
  __shared__ AdmitShared<THREADS, RPT> sm;
  const int tid = threadIdx.x;
  if (tid == 0) block_setup(a, sm);
  __syncthreads();
  const BatchConst b = sm.bc;
  const int64_t tile0 = (int64_t)sm.vb * THREADS * RPT;
  const int64_t nw = sm.nw, row0 = sm.row0;
  const bool entropy = a.p.utility_proxy == GG_UTIL_ENTROPY;
  const int k = KC > 0 ? KC : a.k;
  uint32_t ballots[RPT];
  int my_skip = 0, my_inv = 0;
  unsigned long long my_bad = 0;
#pragma unroll
  for (int j = 0; j < RPT; ++j) {
    const int64_t r = tile0 + (int64_t)j * THREADS + tid;
    const bool in = r < nw;
    const int64_t g = row0 + r;  // trace row
    uint8_t code = GG_DECISION_SKIP;
    if (in) {
      const double* row = a.probs + g * a.stride;
      double xv[KC > 0 ? KC : 16];
      if constexpr (KC == 2) {
        const double2 v = *reinterpret_cast<const double2*>(row);
        xv[0] = v.x; xv[1] = v.y;
      } else if constexpr (KC == 4) {
        const double2 v0 = *reinterpret_cast<const double2*>(row);
        const double2 v1 = *reinterpret_cast<const double2*>(row + 2);
        xv[0] = v0.x; xv[1] = v0.y; xv[2] = v1.x; xv[3] = v1.y;
      } else {
        for (int c = 0; c < k; ++c) xv[c] = row[c];
      }
      double u, jv = 0.0, tau = 0.0;
      bool valid;
      const double now_g = a.now[g];
      int fast = -1;
      if (!a.breakdown) {
        // exact validation (cheap), approximate utility, then the margin test
        bool ok = true, first = true;
        NeumaierSum tot;
        double hf = 0.0, mx = 0.0;
#pragma unroll
        for (int c = 0; c < (KC > 0 ? KC : 16); ++c) {
          if (KC == 0 && c >= k) break;
          const double x = xv[c];
          if (!isfinite(x) || x < 0.0) ok = false;
          tot.add(x);
          if (entropy) hf += entropy_term_fast(x);
          if (first || x > mx) mx = x;
          first = false;
        }
        valid = ok && k >= 2 && !(fabs(f64_sub(tot.result(), 1.0)) > 1e-9);
        if (valid) {
          const double u_f = entropy ? clamp01(-hf / a.ln_k) : f64_sub(1.0, mx);
          fast = decide_fast(a, b, u_f, entropy ? 1e-5 : 0.0, now_g);
          if (fast >= 0) code = (uint8_t)fast;
        }
      }
      if (a.breakdown || (valid && fast < 0)) {
        RowAcc acc;   // exact CPython-order evaluation (controller.py:126-148)
        for (int c = 0; c < k; ++c) acc.add(xv[c], entropy);
        valid = acc.finish(k, entropy, a.ln_k, u);
        if (valid) code = decide_row(a, b, u, now_g, jv, tau);
      }
      if (valid) {
        if (code == GG_DECISION_SKIP) ++my_skip;
      } else {
        code = GG_DECISION_INVALID;
        ++my_inv;
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
    ballots[j] = __ballot_sync(0xffffffffu, in && (code == GG_DECISION_DIRECT || code == GG_DECISION_BATCHED));
  }
  finish_tile<THREADS, RPT>(a, sm, tile0, ballots, my_skip, my_inv, my_bad);
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
  int my_skip = 0, my_inv = 0;
  unsigned long long my_bad = 0;
  if (in) {
    double u = tot_s[lane], jv = 0.0, tau = 0.0;
    if (ok_s[lane]) {
      code = decide_row(a, b, u, a.now[g], jv, tau);
      if (code == GG_DECISION_SKIP) ++my_skip;
    } else {
      code = GG_DECISION_INVALID;
      ++my_inv;
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
  finish_tile<kLargeThreads, 1>(a, sm, tile0, ballots, my_skip, my_inv, my_bad);
}

// K1, large K, fast filter (no breakdown requested; the serving loop): one warp
// per row, coalesced loads, fp64 sum of the probabilities and of fp32-log
// entropy terms, warp reductions — no sequential chain.  A row is recomputed
// exactly (sequential CPython order, one lane) only when its sum lies within
// 1e-13 of the 1e-9 validation bound or J lies within the margin of tau.
__global__ void __launch_bounds__(kLargeThreads) admit_large_fast_kernel(AdmitArgs a) {
  __shared__ AdmitShared<kLargeThreads, 1> sm;
  __shared__ uint8_t codes[kLargeRows];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) block_setup(a, sm);
  __syncthreads();
  const BatchConst b = sm.bc;
  const int64_t tile0 = (int64_t)sm.vb * kLargeRows;
  const int64_t nw = sm.nw, row0 = sm.row0;
  const bool entropy = a.p.utility_proxy == GG_UTIL_ENTROPY;
  for (int lr = warp; lr < kLargeRows; lr += kLargeThreads / 32) {
    const int64_t r = tile0 + lr;
    if (r >= nw) {
      if (lane == 0) codes[lr] = GG_DECISION_SKIP;
      continue;
    }
    const int64_t g = row0 + r;
    const double* row = a.probs + g * a.stride;
    double sum = 0.0, hf = 0.0, mx = -INFINITY;
    bool ok = true;
    for (int c = lane; c < a.k; c += 32) {
      const double x = __ldg(row + c);
      if (!isfinite(x) || x < 0.0) ok = false;
      sum += x;
      if (entropy) hf += entropy_term_fast(x);
      mx = fmax(mx, x);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      sum += __shfl_xor_sync(0xffffffffu, sum, o);
      hf += __shfl_xor_sync(0xffffffffu, hf, o);
      mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    ok = __all_sync(0xffffffffu, ok);
    if (lane == 0) {
      // pairwise-ish fp64 sum of <= K nonnegative terms: |error| < K * 2^-52 * sum
      const double dev = fabs(sum - 1.0), bound = (double)a.k * 2.3e-16 * (sum + 1.0);
      int code;
      bool exact = false, valid = ok && a.k >= 2;
      if (valid && dev > 1e-9 + bound) valid = false;
      else if (valid && dev > 1e-9 - bound) exact = true;   // too close to the bound
      if (valid && !exact) {
        const double u_f = entropy ? clamp01(-hf / a.ln_k) : f64_sub(1.0, mx);
        code = decide_fast(a, b, u_f, entropy ? 1e-5 : 0.0, a.now[g]);
        if (code < 0) exact = true;
      } else {
        code = GG_DECISION_INVALID;
      }
      if (exact) {   // rare: the reference's own sequential evaluation
        RowAcc acc;
        for (int c = 0; c < a.k; ++c) acc.add(row[c], entropy);
        double u, jv, tau;
        code = acc.finish(a.k, entropy, a.ln_k, u) ? decide_row(a, b, u, a.now[g], jv, tau)
                                                   : GG_DECISION_INVALID;
      }
      codes[lr] = (uint8_t)code;
      a.decision[g] = (uint8_t)code;
    }
  }
  __syncthreads();
  const int64_t r = tile0 + tid;           // rows live on warp 0's lanes for the compaction
  const bool in = warp == 0 && r < nw;
  const uint8_t code = in ? codes[tid] : (uint8_t)GG_DECISION_SKIP;
  int my_skip = (in && code == GG_DECISION_SKIP) ? 1 : 0;
  int my_inv = (in && code == GG_DECISION_INVALID) ? 1 : 0;
  unsigned long long my_bad = my_inv ? (unsigned long long)(nw - r) : 0ull;
  uint32_t ballots[1] = {__ballot_sync(0xffffffffu, in && (code == GG_DECISION_DIRECT || code == GG_DECISION_BATCHED))};
  finish_tile<kLargeThreads, 1>(a, sm, tile0, ballots, my_skip, my_inv, my_bad);
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
__global__ void __launch_bounds__(32) outcome_kernel(gg_params p, gg_state* st, const double* lat,
                                                     const double* jou, const int32_t* qd, int64_t n,
                                                     int set_qd, int64_t* err, const double* slots,
                                                     int G, int B, int rank, gg_fifo* fifo) {
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

static int64_t admit_blocks(int64_t n, int32_t k) {
  const int64_t rows_per_block = (k <= 16) ? 256 * 4 : kLargeRows;
  int64_t nb = (n + rows_per_block - 1) / rows_per_block;
  return nb < 1 ? 1 : nb;
}

size_t gg_admit_workspace_bytes(int64_t n) {
  const int64_t nb = (n + kLargeRows - 1) / kLargeRows;  // worst case over kernels
  return kWsHeader + sizeof(unsigned long long) * (size_t)(nb < 1 ? 1 : nb);
}

static int launch_admit(const AdmitArgs& a, void* stream);

// K2 instantiation by window capacity (register slots per lane = ceil(W / 32)).
static int launch_outcome(const gg_params& p, gg_state* st, const double* lat, const double* jou,
                          const int32_t* qd, int64_t n, int set_qd, int64_t* err,
                          const double* slots, int G, int B, int rank, gg_fifo* fifo,
                          void* stream) {
  cudaStream_t s = gg_stream(stream);
  const int w = p.p95_window;
#define GG_OUTCOME(SLOTS) \
  outcome_kernel<SLOTS><<<1, 32, 0, s>>>(p, st, lat, jou, qd, n, set_qd, err, slots, G, B, rank, fifo)
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

static int launch_admit(const AdmitArgs& a, void* stream) {
  const int64_t n = a.n;
  const int32_t k = a.k;
  const double* probs_dev = a.probs;
  const int64_t row_stride = a.stride;
  const int64_t nb = admit_blocks(n, k);
  cudaStream_t s = gg_stream(stream);
  const bool aligned16 = ((reinterpret_cast<uintptr_t>(probs_dev) & 15) == 0) && (row_stride % 2 == 0);
  if (k == 2 && aligned16)
    admit_small_kernel<2, 256, 4><<<(unsigned)nb, 256, 0, s>>>(a);
  else if (k == 4 && aligned16)
    admit_small_kernel<4, 256, 4><<<(unsigned)nb, 256, 0, s>>>(a);
  else if (k <= 16)
    admit_small_kernel<0, 256, 4><<<(unsigned)nb, 256, 0, s>>>(a);
  else if (a.breakdown == nullptr && !getenv("GG_ADMIT_EXACT_ONLY"))
    admit_large_fast_kernel<<<(unsigned)nb, kLargeThreads, 0, s>>>(a);
  else
    admit_large_kernel<<<(unsigned)nb, kLargeThreads, 0, s>>>(a);
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
