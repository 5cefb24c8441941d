"""Columnar trace export (paper_2601_04250_b200.telemetry):
byte-identical to the reference's export_jsonl / export_csv on fixtures written by
the reference itself (tests/golden/make_telemetry_golden.py)."""

from __future__ import annotations

import os
from collections import namedtuple

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _cols():
    z = np.load(os.path.join(GOLD, "telemetry_trace.npz"))
    return {k: z[k] for k in z.files}


def test_jsonl_columns_match_reference_bytes(tmp_path):
    from paper_2601_04250_b200.telemetry import export_jsonl_columns
    out = tmp_path / "t.jsonl"
    export_jsonl_columns(out, **_cols())
    assert out.read_bytes() == open(os.path.join(GOLD, "telemetry_trace.jsonl"), "rb").read()


def test_jsonl_from_records_and_torch_columns(tmp_path):
    import torch
    from paper_2601_04250_b200.telemetry import JSONL_FIELDS, export_jsonl, export_jsonl_columns
    c = _cols()
    want = open(os.path.join(GOLD, "telemetry_trace.jsonl"), "rb").read()
    Rec = namedtuple("Rec", JSONL_FIELDS)
    recs = [Rec(int(c["request_id"][i]), bool(c["admitted"][i]), str(c["path"][i]),
                *(float(c[f][i]) for f in ("enqueue_t", "start_t", "finish_t", "latency_ms", "joules")),
                int(c["predicted_label"][i]), bool(c["correct"][i])) for i in range(len(c["path"]))]
    export_jsonl(type("T", (), {"records": recs})(), tmp_path / "a.jsonl")
    assert (tmp_path / "a.jsonl").read_bytes() == want
    tc = {k: (torch.from_numpy(v) if v.dtype.kind in "fib" else v) for k, v in c.items()}
    export_jsonl_columns(tmp_path / "b.jsonl", **tc)
    assert (tmp_path / "b.jsonl").read_bytes() == want


def test_summary_csv_matches_reference_bytes(tmp_path):
    from paper_2601_04250_b200.telemetry import export_csv
    Row = namedtuple("Row", "label avg_latency_ms std_latency_ms throughput_rps energy_kwh co2_kg "
                            "admitted_count skipped_count accuracy")
    lat0 = float(_cols()["latency_ms"][0])
    rows = [Row("standard", 12.5, 3.25, 401.0, 1.2e-5, 6e-6, 300, 100, 0.9125),
            Row("controlled", lat0, 0.1, float("inf"), 5e-324, 0.0, 0, 400, 1 / 3)]
    export_csv(rows, tmp_path / "s.csv")
    assert (tmp_path / "s.csv").read_bytes() == open(os.path.join(GOLD, "telemetry_summary.csv"), "rb").read()


def test_parallel_chunks_equal_single_process():
    """>= 128 k rows go through the process pool: same bytes as one process and as
    the reference's per-record json.dumps line."""
    import json
    from paper_2601_04250_b200.telemetry import JSONL_FIELDS, jsonl_bytes
    c = _cols()
    reps = (140_000 + len(c["path"]) - 1) // len(c["path"])
    big = {k: np.concatenate([v] * reps) for k, v in c.items()}
    args = [big[f] for f in JSONL_FIELDS]
    par = jsonl_bytes(*args, workers=2)
    one = jsonl_bytes(*args, workers=1)
    assert par == one
    first = json.dumps(dict(zip(JSONL_FIELDS, [a[1].item() if hasattr(a[1], "item") else a[1] for a in args])))
    assert par.splitlines()[1] == first


@pytest.mark.gpu
def test_parallel_export_after_cuda_init():
    """In a process that holds a CUDA context the pool spawns instead of forking."""
    import torch
    from paper_2601_04250_b200.telemetry import JSONL_FIELDS, jsonl_bytes
    torch.zeros(1, device="cuda")
    assert torch.cuda.is_initialized()
    c = _cols()
    reps = (140_000 + len(c["path"]) - 1) // len(c["path"])
    args = [np.concatenate([c[f]] * reps) for f in JSONL_FIELDS]
    assert jsonl_bytes(*args, workers=2) == jsonl_bytes(*args, workers=1)
