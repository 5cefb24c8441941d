"""Loader for the in-tree CUDA library (libgreengate_b200.so, sm_100a).

There is no CPU fallback: if the library is missing or no CUDA device is
present, every compute entry point raises `NativeUnavailable`.  Building the
library (`python -m paper_2601_04250_b200.build`) does not need a GPU.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from . import _abi

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "libgreengate_b200.so")

_P = C.c_void_p
_I64 = C.c_int64
_I32 = C.c_int32
_D = C.c_double

# name -> (restype, argtypes); mirrors include/greengate_b200.h
SIGNATURES: dict[str, tuple] = {
    "gg_version": (C.c_char_p, []),
    "gg_abi_version": (C.c_int, []),
    "gg_state_bytes": (C.c_size_t, []),
    "gg_validate_params": (C.c_int, [_P]),
    "gg_state_init": (C.c_int, [_P, _D, _P]),
    "gg_admit_workspace_bytes": (C.c_size_t, [_I64]),
    "gg_admit": (C.c_int, [_P, _P, _P, _I64, _I32, _I64, _P, _P, _P, _P, _P, _P, _P, C.c_size_t, _P]),
    "gg_outcome": (C.c_int, [_P, _P, _P, _P, _P, _I64, _I32, _P, _P]),
    "gg_reset_clock": (C.c_int, [_P, _D, _P]),
    "gg_set_queue_depth": (C.c_int, [_P, _I32, _P]),
    "gg_epilogue": (C.c_int, [_P, _I64, _I32, _I64, _I32, _P, _P, _P, _P, _P]),
    "gg_utility": (C.c_int, [_P, _I64, _I32, _I64, _I32, _P, _P, _P]),
    "gg_threshold": (C.c_int, [_D, _D, _D, _D, _P, _P, _I64, _P]),
    "gg_cost": (C.c_int, [_D, _D, _D, _P, _P, _I64, _P]),
    # forward pass (include/greengate_b200_forward.h)
    "gg_gemm_bf16": (C.c_int, [_P, _I64, _P, _I64, _P, _I64, _I64, _I64, _I64, _P, _P, _I64, _I32,
                               _I32, _P]),
    "gg_gemm": (C.c_int, [_P, _I64, _P, _I64, _P, _I64, _I64, _I64, _I64, _P, _P]),
    "gg_gemm_ln": (C.c_int, [_P, _I64, _P, _I64, _P, _I64, _I64, _I64, _I64, _P, _P, _P]),
    "gg_streamk_reserve": (C.c_int, []),
    "gg_streamk_mode": (C.c_int, [_I32]),
    "gg_attention": (C.c_int, [_P, _P, _P, _I64, _I32, _I32, _I32, _P, _P]),
    "gg_attention_dep": (C.c_int, [_P, _P, _P, _I64, _I32, _I32, _I32, _P, _P, _P]),
    "gg_gemm_dep": (C.c_int, [_P, _I64, _P, _I64, _P, _I64, _I64, _I64, _I64, _P, _P, _P, _P]),
    "gg_zero_async": (C.c_int, [_P, _I64, _P]),
    "gg_ffn_pair": (C.c_int, [_P, _P, _P, _P, _P, _I64, _I32, _I32, _P, _I32, _P, _P, _P, _P, _P, _P,
                              _P, _P, C.c_float, _P, _P, _P]),
    "gg_step_record_bytes": (C.c_size_t, [_I32, _I32]),
    "gg_publish_step": (C.c_int, [_P, _P, _P, _P, _P, _P, _I32, _I32, _P, _P, _P]),
    "gg_layernorm": (C.c_int, [_P, _I64, _P, _I64, _P, _P, _I64, _I32, C.c_float, _P, _I32, _P]),
    "gg_cls_head": (C.c_int, [_P, _I64, _P, _P, C.c_float, _P, _P, _P, _P, _I32, _P, _I64, _I32,
                              _I32, _P, _P, _P, _P]),
    "gg_cls_head_scratch_bytes": (_I64, [_I32]),
    "gg_set_sm_reserve": (C.c_int, [_I32]),
    "gg_embed_layernorm": (C.c_int, [_P, _P, _P, _P, _P, _P, _I64, _I32, _I32, C.c_float, _P,
                                     _P]),
    "gg_token_gather": (C.c_int, [_P, _P, _I64, _P, _P, _I32, _I32, _P, _P, _P]),
    "gg_conv2d": (C.c_int, [_P, _I32, _I32, _I32, _I32, _P, _I32, _I32, _I32, _I32, _I32, _I32,
                            _P, _P, _I32, _P, _I32, _I32, _P, _P]),
    "gg_conv2d_ds": (C.c_int, [_P, _I32, _I32, _I32, _I32, _P, _I32, _P, _P, _P, _P, _P, _I32, _I32,
                               _P, _P]),
    "gg_conv3x3_shared": (C.c_int, [_P, _I32, _I32, _I32, _I32, _P, _I32, _P, _P, _I32, _P, _P, _P]),
    "gg_conv3x3_padded": (C.c_int, [_P, _I32, _I32, _I32, _I32, _P, _I32, _P, _P, _I32, _P, _P,
                                    _P]),
    "gg_nchw_to_nhwc": (C.c_int, [_P, _I32, _I32, _I32, _I32, _I32, _P, _P]),
    "gg_nchw_to_s2d16": (C.c_int, [_P, _I32, _I32, _I32, _I32, _P, _P]),
    "gg_stem_s2d_span": (C.c_int, [_P, _I32, _I32, _I32, _P, _I32, _P, _I32, _P, _P, _P]),
    "gg_stem_pool_span": (C.c_int, [_P, _I32, _I32, _I32, _P, _I32, _P, _P, _I32, _P, _P]),
    "gg_stem_gather": (C.c_int, [_P, _I64, _P, _P, _I32, _I32, _I32, _P, _P, _I32, _P, _P]),
    "gg_maxpool3x3s2": (C.c_int, [_P, _I32, _I32, _I32, _I32, _P, _I32, _P, _P]),
    "gg_avgpool": (C.c_int, [_P, _I32, _I32, _I32, _P, _I32, _P, _P]),
    "gg_avgpool_fc": (C.c_int, [_P, _I32, _I32, _I32, _I32, _P, _P, _I32, _P, _P, _I64, _P, _P]),
    # serving loop (include/greengate_b200.h)
    "gg_admit_stream": (C.c_int, [_P, _P, _P, _P, _P, _P, _I32, _I64, _P, _I64, _P, _P, _P, _P,
                                  C.c_size_t, _P]),
    "gg_admit_open_stream": (C.c_int, [_P, _P, _P, _P, _P, _I64, _P, _P, _P]),
    "gg_fifo_pop": (C.c_int, [_P, _P, _P, _P, _P, _P, _I32, _P]),
    "gg_fifo_pop_windowed": (C.c_int, [_P, _P, _P, _P, _D, _P, _P, _P, _I32, _P]),
    "gg_fallback_answers": (C.c_int, [_P, _I32, _I64, _P, _P, _P, _P, _I64, _I64, _P, _P, _D, _P,
                                      _P, _P]),
    "gg_served_outcomes": (C.c_int, [_P, _P, _P, _P, _P, _P, _I32, _P]),
    "gg_served_outcomes_trace": (C.c_int, [_P, _P, _P, _P, _P, _P, _P, _P, _I32, _P, _P]),
    "gg_outcome_slots": (C.c_int, [_P, _P, _P, _I32, _I32, _I32, _P, _P, _P]),
    "gg_epilogue_served": (C.c_int, [_P, _P, _I32, _I32, _I64, _P, _P, _P, _P, _P, _P, _P]),
}


class NativeUnavailable(RuntimeError):
    """The sm_100a library or the CUDA device is missing (no CPU fallback)."""


class NativeError(RuntimeError):
    def __init__(self, fn: str, code: int):
        super().__init__(f"{fn} failed with gg_status {code}")
        self.fn = fn
        self.code = code


_lock = threading.Lock()
_lib: C.CDLL | None = None


def load() -> C.CDLL:
    """Load (once) and type the library.  Raises NativeUnavailable if absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise NativeUnavailable(
                f"{LIB_PATH} is missing; build it with `python -m paper_2601_04250_b200.build` "
                "(there is no CPU fallback)")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.gg_abi_version() != _abi.GG_ABI_VERSION:
            raise NativeUnavailable("ABI version mismatch between _abi.py and the library")
        if lib.gg_state_bytes() != _abi.STATE_BYTES:
            raise NativeUnavailable("gg_state layout mismatch between _abi.py and the library")
        _lib = lib
        return lib


def require_cuda():
    """Return torch after checking that a CUDA device is present."""
    import torch

    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device: the greengate B200 path has no CPU fallback")
    load()
    return torch


LAUNCHES = 0  # entry-point calls (each enqueues one kernel); bench.py counts a step with it


def check(fn: str, code: int) -> None:
    global LAUNCHES
    LAUNCHES += 1
    if code != _abi.GG_OK:
        raise NativeError(fn, code)


def ptr(t) -> C.c_void_p | None:
    """Raw device pointer of a torch tensor (None -> NULL)."""
    return None if t is None else C.c_void_p(t.data_ptr())


def stream_ptr(stream=None) -> C.c_void_p:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)
