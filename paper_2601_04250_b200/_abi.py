"""ctypes mirror of include/greengate_b200.h (the C ABI structs and enums).

Kept in lock-step with the header; `tests/test_abi.py` checks sizes/offsets
against the compiled library (`gg_state_bytes`) and against the header text.
"""

from __future__ import annotations

import ctypes as C

GG_ABI_VERSION = 1
GG_P95_WINDOW_MAX = 1024

# gg_status
GG_OK = 0
GG_ERR_INVALID_ARGUMENT = 1
GG_ERR_INVALID_DISTRIBUTION = 2
GG_ERR_NEGATIVE_MEASUREMENT = 3
GG_ERR_INVALID_SCHEDULE = 4
GG_ERR_INVALID_LAMBDA = 5
GG_ERR_CUDA = 6
GG_ERR_UNSUPPORTED = 7

GG_DIR_GEQ, GG_DIR_LT = 0, 1
GG_UTIL_ENTROPY, GG_UTIL_ONE_MINUS_CONFIDENCE = 0, 1
GG_ROUTE_ALL_DIRECT, GG_ROUTE_ALL_BATCHED, GG_ROUTE_THRESHOLD_ON_QUEUE = 0, 1, 2
GG_LATENCY_MODEL, GG_LATENCY_MEASURED, GG_LATENCY_TRACE = 0, 1, 2
GG_DECISION_SKIP, GG_DECISION_DIRECT, GG_DECISION_BATCHED, GG_DECISION_INVALID = 0, 1, 2, 255


class gg_params(C.Structure):
    _fields_ = [
        ("alpha", C.c_double), ("beta", C.c_double), ("gamma", C.c_double),
        ("tau0", C.c_double), ("tau_inf", C.c_double), ("k", C.c_double),
        ("ewma_lambda", C.c_double),
        ("direction", C.c_int32), ("utility_proxy", C.c_int32), ("routing", C.c_int32),
        ("queue_threshold", C.c_int32), ("p95_window", C.c_int32), ("reserved", C.c_int32),
    ]


class gg_channel(C.Structure):
    _fields_ = [("lo", C.c_double), ("hi", C.c_double), ("seen", C.c_int32),
                ("reserved", C.c_int32)]


class gg_state(C.Structure):
    _fields_ = [
        ("n_energy", gg_channel), ("n_queue_depth", gg_channel), ("n_p95_ms", gg_channel),
        ("ewma_joules_per_request", C.c_double), ("total_joules", C.c_double),
        ("t_origin", C.c_double), ("p95_current", C.c_double),
        ("samples_seen", C.c_int64), ("admitted_total", C.c_int64),
        ("skipped_total", C.c_int64), ("outcomes_total", C.c_int64),
        ("queue_depth", C.c_int32), ("win_count", C.c_int32),
        ("win_head", C.c_int32), ("reserved", C.c_int32),
        ("win", C.c_double * GG_P95_WINDOW_MAX),
        ("win_sorted", C.c_double * GG_P95_WINDOW_MAX),
    ]


class gg_snapshot(C.Structure):
    _fields_ = [("queue_depth", C.c_int64), ("p95_latency_ms", C.c_double),
                ("batch_fill", C.c_double)]


class gg_batch_info(C.Structure):
    _fields_ = [("n_admitted", C.c_int64), ("n_skipped", C.c_int64), ("n_invalid", C.c_int64),
                ("first_invalid", C.c_int64), ("energy", C.c_double), ("congestion", C.c_double),
                ("n_decided", C.c_int64), ("snap_queue_depth", C.c_int64),
                ("snap_p95_ms", C.c_double), ("snap_batch_fill", C.c_double)]


class gg_fifo(C.Structure):
    _fields_ = [("head", C.c_int64), ("tail", C.c_int64), ("capacity", C.c_int64),
                ("batch_cap", C.c_int64), ("cursor", C.c_int64), ("trace_len", C.c_int64),
                ("extra_depth", C.c_int64), ("overflow", C.c_int64), ("clock", C.c_double)]


class gg_outcome_model(C.Structure):
    _fields_ = [("batch_base_ms", C.c_double), ("per_item_ms", C.c_double),
                ("batch_base_energy_j", C.c_double), ("per_item_energy_j", C.c_double),
                ("measured_latency", C.c_int32), ("reserved", C.c_int32)]


# Field offsets of gg_state used by the Python shim to read scalars out of the
# device state tensor without copying the 16 KB window.
STATE_OFFSETS = {name: getattr(gg_state, name).offset for name, _ in gg_state._fields_}
STATE_BYTES = C.sizeof(gg_state)
BATCH_INFO_BYTES = C.sizeof(gg_batch_info)
SNAPSHOT_BYTES = C.sizeof(gg_snapshot)


class gg_step_record(C.Structure):
    """gg_step_record (include/greengate_b200.h): header of a published step record."""
    _fields_ = [("count", C.c_int32), ("n_decided", C.c_int32), ("window_start", C.c_int64),
                ("step", C.c_int64), ("reserved", C.c_int64)]
