"""Columnar trace export at 1M scale, byte-identical to the
reference's writers.

The reference serializes a run one record at a time: ``export_jsonl``
(telemetry.py:187-203) builds a dict per ``CompletionRecord`` and calls
``json.dumps`` on it; ``export_csv`` (telemetry.py:148-164) writes summary rows
with ``repr`` floats.  The serving loop here keeps its results as device
columns (decision, prediction, latency, joules, ...), so the export takes
columns: every column is formatted once (``float.__repr__`` over the whole
column — exactly what ``json.dumps`` emits for a finite float — with NaN / ±inf
patched to ``NaN`` / ``Infinity`` / ``-Infinity``, booleans to ``true`` /
``false``, path names JSON-quoted once per distinct value) and the lines are
assembled with one format string.  Same bytes as the reference
(``tests/test_telemetry_export.py`` against fixtures written by the reference
itself); the float repr dominates (~1 us per value in CPython), so at >= 128 k
rows the row range is formatted by a process pool and concatenated in order
(``tools/telemetry_bench.py``: 1 M records, same bytes).  Host-side IO: not a GPU
path.
"""

from __future__ import annotations

import csv
import json
import os
from pathlib import Path
from typing import Iterable, Sequence

import numpy as np

JSONL_FIELDS = ("request_id", "admitted", "path", "enqueue_t", "start_t", "finish_t", "latency_ms",
                "joules", "predicted_label", "correct")
_LINE = ("{{\"request_id\": {}, \"admitted\": {}, \"path\": {}, \"enqueue_t\": {}, \"start_t\": {}, "
         "\"finish_t\": {}, \"latency_ms\": {}, \"joules\": {}, \"predicted_label\": {}, \"correct\": {}}}\n")
CSV_HEADER = ["label", "avg_latency_ms", "std_latency_ms", "throughput_rps", "energy_kwh", "co2_kg",
              "admitted", "skipped", "accuracy"]


def _host(col) -> np.ndarray:
    if hasattr(col, "detach"):          # torch tensor (device or host)
        col = col.detach().cpu().numpy()
    return np.asarray(col)


def _float_tokens(col) -> list[str]:
    """json.dumps' float tokens for a whole column (float.__repr__; NaN / Infinity)."""
    a = np.ascontiguousarray(_host(col), dtype=np.float64)
    toks = list(map(float.__repr__, a.tolist()))
    bad = np.flatnonzero(~np.isfinite(a))
    for i in bad.tolist():
        x = a[i]
        toks[i] = "NaN" if x != x else ("Infinity" if x > 0 else "-Infinity")
    return toks


def _int_tokens(col) -> list[str]:
    return list(map(int.__repr__, _host(col).astype(np.int64).tolist()))


def _bool_tokens(col) -> list[str]:
    return np.where(_host(col).astype(bool), "true", "false").tolist()


def _str_tokens(col) -> list[str]:
    vals = _host(col)
    cache: dict = {}
    out = []
    for v in vals.tolist():
        t = cache.get(v)
        if t is None:
            t = cache[v] = json.dumps(v)
        out.append(t)
    return out


def _chunk_text(cols) -> str:
    request_id, admitted, path, enqueue_t, start_t, finish_t, latency_ms, joules, predicted_label, correct = cols
    toks = (_int_tokens(request_id), _bool_tokens(admitted), _str_tokens(path), _float_tokens(enqueue_t),
            _float_tokens(start_t), _float_tokens(finish_t), _float_tokens(latency_ms), _float_tokens(joules),
            _int_tokens(predicted_label), _bool_tokens(correct))
    return "".join(map(_LINE.format, *toks))


_PAR_MIN = 1 << 17   # rows: below this one process formats everything


def jsonl_bytes(request_id, admitted, path, enqueue_t, start_t, finish_t, latency_ms, joules,
                predicted_label, correct, *, workers: int | None = None) -> str:
    """The text ``export_jsonl`` writes for these records (one line per record).

    Columns are formatted column-at-a-time; at >= 128 k rows the row range is
    split into contiguous chunks formatted by a process pool (``workers``
    processes, default all cores) and concatenated in order — the float repr
    is the cost (~1 us per value in CPython), and it parallelizes perfectly."""
    cols = [_host(c) for c in (request_id, admitted, path, enqueue_t, start_t, finish_t, latency_ms,
                               joules, predicted_label, correct)]
    n = len(cols[0])
    if any(len(c) != n for c in cols):
        raise ValueError("columns must have equal length")
    w = workers if workers is not None else (os.cpu_count() or 1)
    if n < _PAR_MIN or w <= 1:
        return _chunk_text(cols)
    import multiprocessing as mp
    from concurrent.futures import ProcessPoolExecutor
    k = min(w * 4, max(1, n // 32768))
    bounds = [n * i // k for i in range(k + 1)]
    chunks = [[c[bounds[i]:bounds[i + 1]] for c in cols] for i in range(k)]
    # fork is cheap, but not after this process created a CUDA context (the children
    # only format text, yet a forked copy of a CUDA process is unsafe): spawn then
    ctx = "fork"
    try:
        import torch
        if torch.cuda.is_initialized():
            ctx = "spawn"
    except ImportError:
        pass
    with ProcessPoolExecutor(max_workers=w, mp_context=mp.get_context(ctx)) as ex:
        return "".join(ex.map(_chunk_text, chunks))


def export_jsonl_columns(file: str | Path, /, **columns) -> None:
    """export_jsonl (telemetry.py:187-203) from columns named as `JSONL_FIELDS`
    (``path`` is a column — the service path — so the file comes positionally)."""
    missing = [f for f in JSONL_FIELDS if f not in columns]
    if missing:
        raise ValueError(f"missing columns: {missing}")
    text = jsonl_bytes(*(columns[f] for f in JSONL_FIELDS))
    with open(file, "w", newline="") as fh:
        fh.write(text)


def export_jsonl(trace, path: str | Path) -> None:
    """Drop-in for the reference ``export_jsonl(trace, path)``: any object with
    ``.records`` of CompletionRecord-like items."""
    recs = trace.records
    cols = {f: [getattr(r, f) for r in recs] for f in JSONL_FIELDS}
    for f in ("enqueue_t", "start_t", "finish_t", "latency_ms", "joules"):
        cols[f] = np.asarray(cols[f], dtype=np.float64)
    export_jsonl_columns(path, **cols)


def export_csv(rows: Iterable, path: str | Path) -> None:
    """Reference ``export_csv`` (telemetry.py:148-164): summary rows, repr floats."""
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh, lineterminator="\n")
        w.writerow(CSV_HEADER)
        for r in rows:
            w.writerow([r.label, repr(r.avg_latency_ms), repr(r.std_latency_ms), repr(r.throughput_rps),
                        repr(r.energy_kwh), repr(r.co2_kg), r.admitted_count, r.skipped_count,
                        repr(r.accuracy)])


def _ref_line(rec: Sequence) -> str:
    """One record the reference way (for tools/telemetry_bench.py and tests)."""
    return json.dumps(dict(zip(JSONL_FIELDS, rec))) + "\n"


__all__ = ["JSONL_FIELDS", "CSV_HEADER", "jsonl_bytes", "export_jsonl_columns", "export_jsonl", "export_csv"]
