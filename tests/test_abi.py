"""The C-ABI library loads on CPU and exports every symbol include/*.h declares.

No compute call is made here (no GPU); layout checks compare the ctypes mirror
with the compiled library and with the header text.
"""

from __future__ import annotations

import ctypes as C
import glob
import os
import re

import pytest

from paper_2601_04250_b200 import _abi, _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions() -> set[str]:
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        text = open(h).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        for m in re.finditer(r"^[A-Za-z_][\w\s\*]*?\b(gg\w+)\s*\(", text, flags=re.M):
            names.add(m.group(1))
    return names


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(_native.LIB_PATH):
        from paper_2601_04250_b200 import build
        build.build()
    return _native.load()


def test_every_declared_symbol_is_exported(lib):
    names = declared_functions()
    assert len(names) >= 14
    for n in names:
        assert hasattr(lib, n), n
        assert n in _native.SIGNATURES, f"{n} not typed in _native.SIGNATURES"


def test_identity_and_layout(lib):
    assert lib.gg_abi_version() == _abi.GG_ABI_VERSION
    assert lib.gg_state_bytes() == C.sizeof(_abi.gg_state)
    assert b"sm_100a" in lib.gg_version()
    assert lib.gg_admit_workspace_bytes(0) >= 64


def test_param_validation_maps_reference_errors(lib):
    ok = _abi.gg_params(1.0, 0.0, 0.0, 1.0, 0.2, 0.5, 0.9, 0, 0, 0, 4, 100, 0)
    assert lib.gg_validate_params(C.byref(ok)) == _abi.GG_OK
    bad_k = _abi.gg_params(1.0, 0.0, 0.0, 1.0, 0.2, 0.0, 0.9, 0, 0, 0, 4, 100, 0)
    assert lib.gg_validate_params(C.byref(bad_k)) == _abi.GG_ERR_INVALID_SCHEDULE
    bad_lam = _abi.gg_params(1.0, 0.0, 0.0, 1.0, 0.2, 0.5, 1.0, 0, 0, 0, 4, 100, 0)
    assert lib.gg_validate_params(C.byref(bad_lam)) == _abi.GG_ERR_INVALID_LAMBDA
    bad_w = _abi.gg_params(float("inf"), 0.0, 0.0, 1.0, 0.2, 0.5, 0.9, 0, 0, 0, 4, 100, 0)
    assert lib.gg_validate_params(C.byref(bad_w)) == _abi.GG_ERR_INVALID_ARGUMENT
    big_win = _abi.gg_params(1.0, 0.0, 0.0, 1.0, 0.2, 0.5, 0.9, 0, 0, 0, 4, 5000, 0)
    assert lib.gg_validate_params(C.byref(big_win)) == _abi.GG_ERR_INVALID_ARGUMENT


def test_struct_fields_match_header():
    text = open(os.path.join(ROOT, "include", "greengate_b200.h")).read()
    chunk = [c for c in text.split("typedef struct {") if "} gg_state;" in c][0]
    body = chunk.split("} gg_state;")[0]
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    fields = re.findall(r"(\w+)(?:\[[^\]]*\])?\s*;", body)
    assert fields == [f for f, _ in _abi.gg_state._fields_]


def test_product_path_has_no_oracle_import():
    pkg = os.path.join(ROOT, "paper_2601_04250_b200")
    for path in glob.glob(os.path.join(pkg, "**", "*.py"), recursive=True):
        src = open(path).read()
        assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", src, flags=re.M), path
