/*
 * gg_oracle.c — C restatement of the reference admission controller.
 * TEST INFRASTRUCTURE ONLY: loaded by tests/ and by bench.py's cpu_baseline /
 * --impl reference legs as the checker and the CPU baseline; never by the
 * product path.
 *
 * Restates /root/reference/pkg/src/greengate/controller.py:114-358,
 * energy.py:24-87 and telemetry.py:35-46 in plain C with CPython float
 * semantics:
 *   - fp64 throughout, compiled with -ffp-contract=off (no FMA), so every
 *     binary operation rounds like CPython's;
 *   - `sum()` is CPython 3.12's Neumaier-compensated float sum;
 *   - log/exp are glibc's, which is what CPython's math.log/math.exp call.
 * The state and parameter layouts are the ABI structs of include/greengate_b200.h
 * so the device state can be compared field by field.
 * Pinned against the reference by tests/test_oracle.py (golden fixtures made
 * by tests/golden/make_golden.py).
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "../include/greengate_b200.h"

/* CPython 3.12 builtin sum over floats (Objects/bltinmodule.c). */
typedef struct { double s, c; } nsum;
static inline void nsum_add(nsum* a, double x) {
  double t = a->s + x;
  if (fabs(a->s) >= fabs(x)) a->c += (a->s - t) + x;
  else a->c += (x - t) + a->s;
  a->s = t;
}
static inline double nsum_result(const nsum* a) {
  double s = a->s;
  if (a->c != 0.0 && isfinite(a->c)) s += a->c;
  return s;
}
static inline double clamp01(double v) { /* min(1.0, max(0.0, v)) */
  v = (v > 0.0) ? v : 0.0;
  return (v < 1.0) ? v : 1.0;
}

/* _validate_distribution + utility (controller.py:126-148).  Returns 0 on
 * success, -1 on InvalidDistribution. */
static int utility_of(const double* xs, int k, int proxy, double ln_k, double* out) {
  if (k < 2) return -1;
  for (int i = 0; i < k; ++i)
    if (!isfinite(xs[i]) || xs[i] < 0.0) return -1;
  nsum tot = {0.0, 0.0};
  for (int i = 0; i < k; ++i) nsum_add(&tot, xs[i]);
  if (fabs(nsum_result(&tot) - 1.0) > 1e-9) return -1;
  if (proxy == GG_UTIL_ENTROPY) {
    nsum h = {0.0, 0.0};
    for (int i = 0; i < k; ++i)
      if (xs[i] > 0.0) nsum_add(&h, xs[i] * log(xs[i]));
    double hv = -nsum_result(&h);
    *out = clamp01(hv / ln_k);
  } else {
    double m = xs[0];
    for (int i = 1; i < k; ++i)
      if (xs[i] > m) m = xs[i];
    *out = 1.0 - m;
  }
  return 0;
}

static inline void ch_observe(gg_channel* c, double raw) {
  if (!c->seen || raw < c->lo) c->lo = raw;
  if (!c->seen || raw > c->hi) c->hi = raw;
  c->seen = 1;
}
static inline double ch_normalize(gg_channel* c, double raw) {
  ch_observe(c, raw);
  if (c->hi <= c->lo) return 0.0;
  return clamp01((raw - c->lo) / (c->hi - c->lo));
}

static int cmp_double(const void* a, const void* b) {
  double x = *(const double*)a, y = *(const double*)b;
  return (x > y) - (x < y);
}

/* percentile_nearest_rank(window, 95.0) (telemetry.py:35-46). */
static double window_p95(const gg_state* s, int cap) {
  if (s->win_count == 0) return 0.0;
  double tmp[GG_P95_WINDOW_MAX];
  for (int i = 0; i < s->win_count; ++i) tmp[i] = s->win[(s->win_head + i) % cap];
  qsort(tmp, (size_t)s->win_count, sizeof(double), cmp_double);
  double rank = ceil(95.0 / 100.0 * (double)s->win_count);
  return tmp[(int)rank - 1];
}

void ggo_state_init(gg_state* s, double t_origin) {
  memset(s, 0, sizeof(*s));
  s->t_origin = t_origin;
}

/* Sequential decide() over n rows against one frozen snapshot
 * (controller.py:309-343).  snapshot == NULL -> default snapshot
 * (controller.py:295-300; queue depth = state.queue_depth as in the gateway). */
void ggo_admit(const gg_params* p, gg_state* s, const double* probs, long n, int k,
               long stride, const double* now, const gg_snapshot* snapshot,
               unsigned char* decision, double* breakdown, int* admitted_idx,
               gg_batch_info* info) {
  const double ln_k = log((double)k);
  gg_snapshot snap;
  if (snapshot) snap = *snapshot;
  else { snap.queue_depth = s->queue_depth; snap.p95_latency_ms = s->p95_current; snap.batch_fill = 0.0; }
  long n_adm = 0, n_skip = 0, n_inv = 0, first_bad = -1;
  double e_last = 0.0, c_last = 0.0;
  for (long i = 0; i < n; ++i) {
    double u;
    if (utility_of(probs + i * stride, k, p->utility_proxy, ln_k, &u) != 0) {
      decision[i] = GG_DECISION_INVALID;
      if (first_bad < 0) first_bad = i;
      ++n_inv;
      if (breakdown) { breakdown[3 * i] = NAN; breakdown[3 * i + 1] = NAN; breakdown[3 * i + 2] = NAN; }
      continue;
    }
    double e = 0.0;
    if (s->samples_seen > 0) e = ch_normalize(&s->n_energy, s->ewma_joules_per_request);
    double c = (ch_normalize(&s->n_queue_depth, (double)snap.queue_depth)
                + ch_normalize(&s->n_p95_ms, snap.p95_latency_ms) + snap.batch_fill) / 3.0;
    double j = p->alpha * u + p->beta * e + p->gamma * c;
    double el = now[i] - s->t_origin;
    el = (el > 0.0) ? el : 0.0;
    double tau = p->tau_inf + (p->tau0 - p->tau_inf) * exp(-p->k * el);
    int adm = (p->direction == GG_DIR_GEQ) ? (j >= tau) : (j < tau);
    unsigned char code = GG_DECISION_SKIP;
    if (adm) {
      if (p->routing == GG_ROUTE_ALL_BATCHED) code = GG_DECISION_BATCHED;
      else if (p->routing == GG_ROUTE_THRESHOLD_ON_QUEUE)
        code = (snap.queue_depth > p->queue_threshold) ? GG_DECISION_BATCHED : GG_DECISION_DIRECT;
      else code = GG_DECISION_DIRECT;
      if (admitted_idx) admitted_idx[n_adm] = (int)i;
      ++n_adm;
      s->admitted_total += 1;
    } else {
      ++n_skip;
      s->skipped_total += 1;
    }
    decision[i] = code;
    if (breakdown) { breakdown[3 * i] = u; breakdown[3 * i + 1] = j; breakdown[3 * i + 2] = tau; }
    e_last = e; c_last = c;
  }
  if (info) {
    info->n_admitted = n_adm; info->n_skipped = n_skip; info->n_invalid = n_inv;
    info->first_invalid = first_bad; info->energy = e_last; info->congestion = c_last;
    info->n_decided = n; info->snap_queue_depth = snap.queue_depth;
    info->snap_p95_ms = snap.p95_latency_ms; info->snap_batch_fill = snap.batch_fill;
  }
}

/* record_outcome() x n in order (controller.py:345-358).  Returns the index of
 * the first negative measurement (which is not applied) or -1. */
long ggo_outcome(const gg_params* p, gg_state* s, const double* lat, const double* joules,
                 const int* qd, long n, int set_queue_depth) {
  const int cap = p->p95_window;
  for (long i = 0; i < n; ++i) {
    if (lat[i] < 0.0 || joules[i] < 0.0 || qd[i] < 0) return i;
    /* EnergyLedger.observe_request -> ewma_update (energy.py:24-36, 75-87) */
    if (s->samples_seen > 0)
      s->ewma_joules_per_request = p->ewma_lambda * s->ewma_joules_per_request
                                   + (1.0 - p->ewma_lambda) * joules[i];
    else
      s->ewma_joules_per_request = joules[i];
    s->samples_seen += 1;
    s->total_joules += joules[i];
    /* deque(maxlen=p95_window).append */
    if (s->win_count < cap) {
      s->win[(s->win_head + s->win_count) % cap] = lat[i];
      s->win_count += 1;
    } else {
      s->win[s->win_head] = lat[i];
      s->win_head = (s->win_head + 1) % cap;
    }
    s->p95_current = window_p95(s, cap);
    ch_observe(&s->n_energy, s->ewma_joules_per_request);
    ch_observe(&s->n_queue_depth, (double)qd[i]);
    ch_observe(&s->n_p95_ms, s->p95_current);
    s->outcomes_total += 1;
    if (set_queue_depth) s->queue_depth = qd[i];
  }
  return -1;
}

/* Epilogue oracle: fp32 logits -> fp64 probs, first-max argmax. */
void ggo_softmax(const float* logits, long n, int k, double* probs, int* argmax) {
  for (long i = 0; i < n; ++i) {
    const float* x = logits + i * k;
    double m = (double)x[0];
    for (int j = 1; j < k; ++j) if ((double)x[j] > m) m = (double)x[j];
    double s = 0.0;
    for (int j = 0; j < k; ++j) { double v = exp((double)x[j] - m); probs[i * k + j] = v; s += v; }
    int am = 0; double best = -1.0;
    for (int j = 0; j < k; ++j) {
      probs[i * k + j] /= s;
      if (probs[i * k + j] > best) { best = probs[i * k + j]; am = j; }
    }
    argmax[i] = am;
  }
}
