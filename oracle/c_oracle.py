"""ctypes loader for the C restatement (oracle/gg_oracle.c) — TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs use this,
as the checker / CPU baseline.  numpy arrays in, numpy arrays out.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from paper_2601_04250_b200 import _abi

from . import build as _build

_lib = None


def lib():
    global _lib
    if _lib is None:
        path = _build.LIB
        if not os.path.exists(path):
            path = _build.build()
        L = C.CDLL(path)
        P = C.c_void_p
        L.ggo_state_init.argtypes = [P, C.c_double]
        L.ggo_admit.argtypes = [P, P, P, C.c_long, C.c_int, C.c_long, P, P, P, P, P, P]
        L.ggo_outcome.argtypes = [P, P, P, P, P, C.c_long, C.c_int]
        L.ggo_outcome.restype = C.c_long
        L.ggo_softmax.argtypes = [P, C.c_long, C.c_int, P, P]
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


class COracle:
    """One controller replica on the host (state = a gg_state struct)."""

    def __init__(self, params: _abi.gg_params, t_origin: float = 0.0):
        self.params = params
        self.state = _abi.gg_state()
        lib().ggo_state_init(C.byref(self.state), C.c_double(t_origin))

    def admit(self, probs: np.ndarray, now: np.ndarray, snapshot=None, want_breakdown=True):
        probs = np.ascontiguousarray(probs, dtype=np.float64)
        now = np.ascontiguousarray(now, dtype=np.float64)
        n, k = probs.shape
        dec = np.empty(n, np.uint8)
        bd = np.empty((n, 3), np.float64) if want_breakdown else None
        idx = np.empty(n, np.int32)
        info = _abi.gg_batch_info()
        snap = None
        if snapshot is not None:
            snap = _abi.gg_snapshot(int(snapshot[0]), float(snapshot[1]), float(snapshot[2]))
        lib().ggo_admit(C.byref(self.params), C.byref(self.state), _ptr(probs), n, k, k,
                        _ptr(now), C.byref(snap) if snap is not None else None,
                        _ptr(dec), _ptr(bd), _ptr(idx), C.byref(info))
        return dec, bd, idx[: info.n_admitted].copy(), info

    def outcome(self, lat, joules, qd, set_queue_depth=False) -> int:
        lat = np.ascontiguousarray(lat, dtype=np.float64)
        joules = np.ascontiguousarray(joules, dtype=np.float64)
        qd = np.ascontiguousarray(qd, dtype=np.int32)
        return int(lib().ggo_outcome(C.byref(self.params), C.byref(self.state), _ptr(lat),
                                     _ptr(joules), _ptr(qd), len(lat), int(set_queue_depth)))


def softmax(logits: np.ndarray):
    logits = np.ascontiguousarray(logits, dtype=np.float32)
    n, k = logits.shape
    probs = np.empty((n, k), np.float64)
    am = np.empty(n, np.int32)
    lib().ggo_softmax(_ptr(logits), n, k, _ptr(probs), _ptr(am))
    return probs, am
