/*
 * greengate_b200.h — C ABI of the B200-native gated-inference hot path.
 *
 * This is the drop-in boundary.  The reference `greengate`
 * package is pure Python; its de-facto operator interface for this path is the
 * `AdmissionController` object (pkg/src/greengate/controller.py:256-362).  The
 * Python shim in `paper_2601_04250_b200/controller.py` keeps that object's
 * names, arguments and exceptions and calls the entry points below through
 * ctypes (INTEGRATION.md shows the binding).  Each entry point names the
 * reference interface it replaces.
 *
 * Conventions
 *   - plain pointers and sizes only; no torch types;
 *   - every `*_dev` pointer is CUDA device memory owned by the caller
 *     (the library never allocates or frees device memory);
 *   - every compute call is stream-ordered on `stream` (a cudaStream_t passed
 *     as void*) and returns immediately; device-side per-row errors are
 *     reported in caller-provided device buffers;
 *   - the return value is a gg_status for launch/argument errors only.
 *
 * Numerics: all controller arithmetic is IEEE fp64, evaluated in the
 * reference's operation order with no FMA contraction, CPython-3.12
 * Neumaier summation for `sum()`, and ln(K) computed on the host with libm.
 */
#ifndef GREENGATE_B200_H
#define GREENGATE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GG_ABI_VERSION 1
/* Largest supported p95 latency window (reference default 100,
 * controller.py:274 / servesim.py:80). */
#define GG_P95_WINDOW_MAX 1024

typedef enum {
  GG_OK = 0,
  GG_ERR_INVALID_ARGUMENT = 1,     /* ValueError / ConfigError */
  GG_ERR_INVALID_DISTRIBUTION = 2, /* errors.py:8  InvalidDistribution */
  GG_ERR_NEGATIVE_MEASUREMENT = 3, /* errors.py:20 NegativeMeasurement */
  GG_ERR_INVALID_SCHEDULE = 4,     /* errors.py:12 InvalidSchedule */
  GG_ERR_INVALID_LAMBDA = 5,       /* errors.py:16 InvalidLambda */
  GG_ERR_CUDA = 6,                 /* launch failure */
  GG_ERR_UNSUPPORTED = 7
} gg_status;

/* Direction (controller.py:38-47) */
enum { GG_DIR_GEQ = 0, GG_DIR_LT = 1 };
/* UtilityProxy (controller.py:50-52) */
enum { GG_UTIL_ENTROPY = 0, GG_UTIL_ONE_MINUS_CONFIDENCE = 1 };
/* RoutePolicy (controller.py:55-58) */
enum { GG_ROUTE_ALL_DIRECT = 0, GG_ROUTE_ALL_BATCHED = 1, GG_ROUTE_THRESHOLD_ON_QUEUE = 2 };
/* Per-row decision codes written by gg_admit (AdmissionDecision.admit/path,
 * controller.py:206-211; ServicePath controller.py:61-64). */
enum {
  GG_DECISION_SKIP = 0,        /* admit=False, path=NONE */
  GG_DECISION_DIRECT = 1,      /* admit=True,  path=DIRECT */
  GG_DECISION_BATCHED = 2,     /* admit=True,  path=BATCHED */
  GG_DECISION_INVALID = 255    /* InvalidDistribution: no state change */
};

/* Immutable controller parameters: CostWeights (controller.py:73-88),
 * ThresholdSchedule minus t_origin (controller.py:91-111), the rest of
 * ControllerConfig (controller.py:219-233), EnergyLedger.ewma_lambda
 * (energy.py:60) and the p95 window length (controller.py:274). */
typedef struct {
  double alpha, beta, gamma;
  double tau0, tau_inf, k;
  double ewma_lambda;
  int32_t direction;
  int32_t utility_proxy;
  int32_t routing;
  int32_t queue_threshold;
  int32_t p95_window;
  int32_t reserved;
} gg_params;

/* One NormalizerChannel (controller.py:157-183).  `seen` = 0 stands for the
 * reference's running_min/running_max being None. */
typedef struct {
  double lo, hi;
  int32_t seen;
  int32_t reserved;
} gg_channel;

/* Mutable loop state, resident in device memory (one per controller).
 * Mirrors AdmissionController fields (controller.py:276-287) plus the
 * EnergyLedger EWMA (energy.py:55-87).  The latency window is kept twice: in
 * arrival order (the deque, controller.py:285) and sorted, so the nearest-rank
 * p95 (telemetry.py:35-46) is an O(1) read. */
typedef struct {
  gg_channel n_energy;       /* NormalizerState.energy      */
  gg_channel n_queue_depth;  /* NormalizerState.queue_depth */
  gg_channel n_p95_ms;       /* NormalizerState.p95_ms      */
  double ewma_joules_per_request;
  double total_joules;
  double t_origin;           /* ThresholdSchedule.t_origin; reset_clock mutates it */
  double p95_current;        /* p95 of the window, 0.0 when empty (controller.py:289-293) */
  int64_t samples_seen;
  int64_t admitted_total;
  int64_t skipped_total;
  int64_t outcomes_total;
  int32_t queue_depth;       /* last reported depth (gateway.py:50, 191, 230) */
  int32_t win_count;         /* len(deque) */
  int32_t win_head;          /* index of the oldest element in win[] */
  int32_t reserved;
  double win[GG_P95_WINDOW_MAX];        /* circular, arrival order */
  double win_sorted[GG_P95_WINDOW_MAX]; /* first win_count entries ascending */
} gg_state;

/* CongestionSnapshot (servesim.py:113-119). */
typedef struct {
  int64_t queue_depth;
  double p95_latency_ms;
  double batch_fill;
} gg_snapshot;

/* Per-launch summary written by gg_admit (device memory). */
typedef struct {
  int64_t n_admitted;
  int64_t n_skipped;
  int64_t n_invalid;
  int64_t first_invalid;     /* -1 when every row is valid */
  double energy;             /* E(x), identical for every valid row of the batch */
  double congestion;         /* C(x), identical for every valid row of the batch */
  int64_t n_decided;         /* rows decided by this launch */
  int64_t snap_queue_depth;  /* the snapshot the batch was decided against */
  double snap_p95_ms;
  double snap_batch_fill;
} gg_batch_info;

/* ---- library identity ---------------------------------------------------- */
const char* gg_version(void);
int gg_abi_version(void);
size_t gg_state_bytes(void);
/* Replaces EnergyLedger(ewma_lambda) + ControllerConfig.build(...) state setup
 * (controller.py:235-287; energy.py:55-73): validates params, zeroes state,
 * sets t_origin.  Returns GG_ERR_INVALID_SCHEDULE / GG_ERR_INVALID_LAMBDA like
 * ThresholdSchedule.__post_init__ (controller.py:100-105) and
 * EnergyLedger.__post_init__ (energy.py:64-69). */
int gg_validate_params(const gg_params* params);
int gg_state_init(gg_state* state_dev, double t_origin, void* stream);

/* ---- K1: fused admission + order-preserving compaction -------------------- */
/* Replaces AdmissionController.decide (controller.py:309-343) applied to the
 * rows of `probs_dev` in order against ONE congestion snapshot (the frozen
 * snapshot of a micro-batch; with n == 1 it is exactly one decide() call).
 *   probs_dev      [n, row_stride] fp64, first k columns are the scores
 *   now_dev        [n] fp64 decision time per row (controller.py:327)
 *   snapshot_dev   NULL -> the default snapshot (queue_depth from state,
 *                  state p95, batch_fill 0; controller.py:295-300)
 *   decision_dev   [n] u8 GG_DECISION_* codes
 *   breakdown_dev  NULL or [n, 3] fp64 (utility, composite, threshold)
 *   admitted_idx_dev NULL or [n] int32: ascending indices of admitted rows
 *   info_dev       gg_batch_info (device)
 *   workspace_dev  >= gg_admit_workspace_bytes(n) bytes, zero-filled before
 *                  first use; every launch leaves it zero-filled again
 * Effects on state (stream-ordered): admitted_total/skipped_total += counts;
 * the queue/p95 (and energy) normalizer channels observe the snapshot if at
 * least one row was valid — exactly what sequential decide() calls do. */
size_t gg_admit_workspace_bytes(int64_t n);
int gg_admit(const gg_params* params, gg_state* state_dev,
             const double* probs_dev, int64_t n, int32_t k, int64_t row_stride,
             const double* now_dev, const gg_snapshot* snapshot_dev,
             uint8_t* decision_dev, double* breakdown_dev,
             int32_t* admitted_idx_dev, gg_batch_info* info_dev,
             void* workspace_dev, size_t workspace_bytes, void* stream);

/* ---- K2: outcome feedback -------------------------------------------------- */
/* Replaces AdmissionController.record_outcome (controller.py:345-358) for n
 * served requests in completion order: EWMA (energy.py:24-36, 75-87), latency
 * window + nearest-rank p95 (controller.py:285, 289-293), channel observes.
 * A negative value stops the sequence at that index (earlier outcomes stay
 * applied, like a Python loop that raises) and writes the index to
 * error_index_dev (else -1).  queue_depth of the last applied outcome becomes
 * state.queue_depth when `set_queue_depth` != 0 (gateway.py:230). */
int gg_outcome(const gg_params* params, gg_state* state_dev,
               const double* latency_ms_dev, const double* joules_dev,
               const int32_t* queue_depth_dev, int64_t n, int32_t set_queue_depth,
               int64_t* error_index_dev, void* stream);

/* Replaces AdmissionController.reset_clock (controller.py:360-362). */
int gg_reset_clock(gg_state* state_dev, double t_origin, void* stream);
/* Sets the externally reported queue depth (gateway.py:191-192). */
int gg_set_queue_depth(gg_state* state_dev, int32_t queue_depth, void* stream);

/* ---- K3: logit -> probability epilogue ------------------------------------ */
/* fp32 logits [n, k] (row stride ld) -> fp64 softmax probabilities that pass
 * _validate_distribution (controller.py:126-135), first-max argmax
 * (RequestFeatures.top_class, workload.py:42-43), confidence (max p) and the
 * controller's utility of the row (entropy_utility controller.py:138-142 or
 * one_minus_confidence_utility 145-148).  Any output pointer may be NULL. */
int gg_epilogue(const float* logits_dev, int64_t n, int32_t k, int64_t ld,
                int32_t utility_proxy, double* probs_dev, int32_t* argmax_dev,
                double* confidence_dev, double* utility_dev, void* stream);

/* ---- serving loop: device FIFO between admission and the forward --------- */
/* The admitted requests of every admission window are appended (in trace
 * order) to a device ring; each forward step pops up to batch_cap of them.
 * The ring depth is the queue depth of the congestion snapshot and
 * depth / batch_cap its batch fill (servesim.py:208-220 semantics), so the
 * whole closed loop runs without a host round-trip. */
typedef struct {
  int64_t head;         /* requests popped into forward batches */
  int64_t tail;         /* requests admitted */
  int64_t capacity;     /* ring slots, power of two */
  int64_t batch_cap;    /* forward batch size B */
  int64_t cursor;       /* next trace row to decide */
  int64_t trace_len;    /* rows of the resident trace */
  int64_t extra_depth;  /* queue depth of the other ranks (multi-GPU exchange) */
  int64_t overflow;     /* admissions lost to a full ring (must stay 0) */
  double clock;         /* trace time of the last pop (gg_fifo_pop_windowed), monotone */
} gg_fifo;

/* Stream form of gg_admit: decides rows [fifo.cursor, fifo.cursor + window)
 * of a device-resident trace (probs [trace_len, row_stride], now [trace_len]),
 * writes decision_dev[row] (trace indexed), appends admitted rows to the ring
 * (ids + admission timestamps), advances cursor/tail.  snapshot_dev NULL ->
 * snapshot from the FIFO: queue_depth = tail - head + extra_depth, p95 from
 * state, batch_fill = min(1, (tail - head) / batch_cap). */
int gg_admit_stream(const gg_params* params, gg_state* state_dev, gg_fifo* fifo_dev,
                    int32_t* ring_ids_dev, uint64_t* ring_ns_dev, const double* probs_dev,
                    int32_t k, int64_t row_stride, const double* now_dev, int64_t window,
                    const gg_snapshot* snapshot_dev, uint8_t* decision_dev,
                    gg_batch_info* info_dev, void* workspace_dev, size_t workspace_bytes,
                    void* stream);
/* Open-loop arm of Simulation._decide (servesim.py:231-240, controller
 * disabled): every row of the window [fifo.cursor, +window) is admitted with
 * the static route (ALL_DIRECT -> DIRECT, ALL_BATCHED -> BATCHED,
 * THRESHOLD_ON_QUEUE -> BATCHED iff depth + extra_depth > queue_threshold) and
 * appended to the ring; no score is read or validated.  The state gets the
 * counters and snapshot observes of an always-admitting decide(). */
int gg_admit_open_stream(const gg_params* params, gg_state* state_dev, gg_fifo* fifo_dev,
                         int32_t* ring_ids_dev, uint64_t* ring_ns_dev, int64_t window,
                         uint8_t* decision_dev, gg_batch_info* info_dev, void* stream);
/* Pops n = min(B, depth) requests: batch_ids[0..n) (trace rows), batch_ns,
 * *count_dev = n. */
int gg_fifo_pop(gg_fifo* fifo_dev, const int32_t* ring_ids_dev, const uint64_t* ring_ns_dev,
                int32_t* batch_ids_dev, uint64_t* batch_ns_dev, int32_t* count_dev, int32_t B,
                void* stream);
/* Path-B pop with the reference's flush policy (batch_flush_policy,
 * servesim.py:148-162): with batching_window_s > 0 the batch flushes when B
 * requests are pending (n = B) or the oldest has waited >= window - 1e-12 s of
 * trace time (n = depth), else n = 0.  The trace clock is now_dev[cursor - 1]
 * (the last decided arrival); once the trace is exhausted the batch timer
 * fires (clock = oldest arrival + window).  fifo.clock records it.
 * batching_window_s == 0: size trigger only (n = min(B, depth)). */
int gg_fifo_pop_windowed(gg_fifo* fifo_dev, const int32_t* ring_ids_dev,
                         const uint64_t* ring_ns_dev, const double* now_dev,
                         double batching_window_s, int32_t* batch_ids_dev,
                         uint64_t* batch_ns_dev, int32_t* count_dev, int32_t B, void* stream);
/* Fallback answers and accounting (Simulation._complete, servesim.py:246-256)
 * for the rows a window decided (fifo_dev/info_dev: the rows gg_admit_stream
 * just decided; else [row0, row0 + n)): answer[row] = top_class(scores)
 * (first max, workload.py:42-43) for every decided row; correct[row] =
 * (top == label) for admitted rows, and (top == label AND coin >= degradation)
 * for skipped rows, where coins_dev is the host-drawn `_fb_rng` stream consumed
 * in trace order by the skipped rows with top == label (*coin_cursor_dev
 * advances).  Invalid rows (255) are left untouched. */
int gg_fallback_answers(const double* probs_dev, int32_t k, int64_t row_stride,
                        const int32_t* labels_dev, const uint8_t* decision_dev,
                        const gg_fifo* fifo_dev, const gg_batch_info* info_dev, int64_t row0,
                        int64_t n, const double* coins_dev, int64_t* coin_cursor_dev,
                        double fallback_degradation, int32_t* answer_dev, uint8_t* correct_dev,
                        void* stream);
/* Outcome model of a served batch (servesim.py:137-139, 303-305 for the
 * modeled path; %globaltimer latency for the measured path). */
enum {
  GG_LATENCY_MODEL = 0,     /* latency = base + per_item * n (service time only) */
  GG_LATENCY_MEASURED = 1,  /* device %globaltimer: completion - admission */
  GG_LATENCY_TRACE = 2      /* trace time: (fifo.clock + service_s - arrival) * 1000,
                               the reference's finish_t - enqueue_t (servesim.py:258-266) */
};
typedef struct {
  double batch_base_ms, per_item_ms;        /* modeled latency = base + per_item * n */
  double batch_base_energy_j, per_item_energy_j;  /* joules each = (base + per_item*n)/n */
  int32_t measured_latency;                 /* GG_LATENCY_* */
  int32_t reserved;
} gg_outcome_model;
/* Writes one rank's step into its exchange slot (fp64, GG_SLOT_LEN(B) values):
 *   [0, B)      latency_ms of the served requests
 *   [B, 2B)     joules
 *   [2B, 3B)    queue depth reported with each outcome
 *   3B + 0..7   n_served, fifo depth after the pop, and the admission effects
 *               of this step (n_decided, n_invalid, n_admitted, n_skipped,
 *               snapshot queue depth, snapshot p95) copied from info_dev. */
#define GG_SLOT_LEN(B) (3 * (B) + 8)
int gg_served_outcomes(const gg_fifo* fifo_dev, const int32_t* count_dev,
                       const uint64_t* batch_ns_dev, const gg_outcome_model* model,
                       const gg_batch_info* info_dev, double* slot_dev, int32_t B, void* stream);
/* Same, with the served batch's trace rows and arrival times (needed by
 * GG_LATENCY_TRACE); latency_row_dev (NULL or fp64 [trace_len]) receives each
 * served request's latency_ms at its trace row (CompletionRecord.latency_ms). */
/* Step record written straight into pinned (host-mapped) memory by the serving
 * step's last kernel, in place of device -> host copies: the served batch's
 * predictions / confidences and the window's decisions.  Two slots alternate
 * by the device step counter *seq_dev (slot = seq & 1, then seq + 1), so the
 * host reads step i's record while step i + 1 runs.  Layout of one slot
 * (gg_step_record_bytes(B, W) bytes): the header, int32 pred[B], double
 * conf[B] (8-byte aligned), uint8 decision[W]. */
typedef struct {
  int32_t count;         /* requests served by the step */
  int32_t n_decided;     /* window rows decided by the step */
  int64_t window_start;  /* trace row of the window's first decision */
  int64_t step;          /* the device step counter before this step */
  int64_t reserved;
} gg_step_record;
size_t gg_step_record_bytes(int32_t B, int32_t W);
int gg_publish_step(const int32_t* count_dev, const int32_t* batch_pred_dev,
                    const double* batch_conf_dev, const uint8_t* decision_dev,
                    const gg_batch_info* info_dev, const gg_fifo* fifo_dev, int32_t B, int32_t W,
                    void* host_records, int64_t* seq_dev, void* stream);

int gg_served_outcomes_trace(const gg_fifo* fifo_dev, const int32_t* count_dev,
                             const uint64_t* batch_ns_dev, const int32_t* batch_ids_dev,
                             const double* now_dev, const gg_outcome_model* model,
                             const gg_batch_info* info_dev, double* slot_dev, int32_t B,
                             double* latency_row_dev, void* stream);
/* Applies G exchange slots (all-reduced) to this rank's replica: first the
 * other ranks' admission effects (normalizer observes of their snapshots,
 * counters), then every rank's outcomes in rank order (K2, record_outcome
 * semantics); sets fifo.extra_depth = sum of the other ranks' depths.  Every
 * rank applies the same slots, so replicas stay bit-identical. */
int gg_outcome_slots(const gg_params* params, gg_state* state_dev, const double* slots_dev,
                     int32_t G, int32_t B, int32_t rank, gg_fifo* fifo_dev,
                     int64_t* error_index_dev, void* stream);
/* K3 for a served batch: logits [B, ld] fp32 (first *count_dev rows valid) ->
 * predicted[batch_ids[i]] (first max), confidence[batch_ids[i]] (fp64 max p),
 * optionally fp64 probabilities [B, k] and batch-local copies
 * batch_predicted[i] / batch_confidence[i] (for a compact device->host read).
 * k <= 1024 (GG_ERR_UNSUPPORTED otherwise). */
int gg_epilogue_served(const float* logits_dev, const int32_t* count_dev, int32_t B, int32_t k,
                       int64_t ld, const int32_t* batch_ids_dev, int32_t* predicted_dev,
                       double* confidence_dev, double* probs_dev, int32_t* batch_predicted_dev,
                       double* batch_confidence_dev, void* stream);

/* ---- stateless batch forms of the controller's pure functions ------------- */
/* entropy_utility / one_minus_confidence_utility (controller.py:138-148) over
 * n rows: utility_dev[i] (NaN when invalid), valid_dev[i] = 0 when the row
 * would raise InvalidDistribution (controller.py:126-135). */
int gg_utility(const double* probs_dev, int64_t n, int32_t k, int64_t row_stride,
               int32_t utility_proxy, double* utility_dev, uint8_t* valid_dev, void* stream);
/* threshold_at (controller.py:114-123) for n times against one schedule. */
int gg_threshold(double tau0, double tau_inf, double k, double t_origin,
                 const double* t_dev, double* tau_dev, int64_t n, void* stream);
/* cost (controller.py:214-216) for n (u, e, c) triples, [n, 3] row-major. */
int gg_cost(double alpha, double beta, double gamma, const double* uec_dev,
            double* j_dev, int64_t n, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* GREENGATE_B200_H */
