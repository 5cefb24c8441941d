"""Golden bytes of the REFERENCE trace writers (build container only).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_telemetry_golden.py

Builds CompletionRecords (random plus edge values: -0.0, subnormal, 1e16, 1e-5,
NaN, +-inf, large ints, all three paths) and SummaryRows, writes them with the
reference's own ``export_jsonl`` / ``export_csv`` (pkg/src/greengate/
telemetry.py) and stores the columns (.npz) and the exact output bytes next to
this script.  Nothing at test time reads /root/reference.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from greengate.servesim import CompletionRecord, RunTrace  # noqa: E402
from greengate.telemetry import SummaryRow, export_csv, export_jsonl  # noqa: E402


def main():
    rng = np.random.default_rng(20260101)
    n = 400
    paths = np.array(["DIRECT", "BATCHED", "NONE"])[rng.integers(0, 3, n)]
    enq = np.cumsum(rng.exponential(0.01, n))
    start = enq + rng.exponential(0.002, n)
    fin = start + rng.exponential(0.02, n)
    lat = (fin - enq) * 1e3
    jl = rng.random(n) * 5.0
    special = [0.0, -0.0, 5e-324, 1e16, 1e-5, 1.0000000000000002, float("nan"), float("inf"),
               float("-inf"), 123456789.123456789, 1e-4, 0.1]
    for i, v in enumerate(special):
        lat[10 + i] = v
        jl[30 + i] = v
    rid = np.arange(n, dtype=np.int64) * 7919 + (1 << 40)
    adm = paths != "NONE"
    pred = rng.integers(-1, 1000, n)
    cor = rng.random(n) < 0.5
    recs = [CompletionRecord(int(rid[i]), bool(adm[i]), str(paths[i]), float(enq[i]), float(start[i]),
                             float(fin[i]), float(lat[i]), float(jl[i]), int(pred[i]), bool(cor[i]))
            for i in range(n)]
    trace = RunTrace(records=recs, makespan_s=float(fin[-1]), ledger=None, admitted=int(adm.sum()),
                     skipped=int((~adm).sum()))
    export_jsonl(trace, os.path.join(HERE, "telemetry_trace.jsonl"))
    np.savez(os.path.join(HERE, "telemetry_trace.npz"), request_id=rid, admitted=adm, path=paths,
             enqueue_t=enq, start_t=start, finish_t=fin, latency_ms=lat, joules=jl,
             predicted_label=pred, correct=cor)
    rows = [SummaryRow("standard", 12.5, 3.25, 401.0, 1.2e-5, 6e-6, 300, 100, 0.9125),
            SummaryRow("controlled", float(lat[0]), 0.1, float("inf"), 5e-324, 0.0, 0, 400, 1 / 3)]
    export_csv(rows, os.path.join(HERE, "telemetry_summary.csv"))
    print("wrote telemetry_trace.jsonl / .npz, telemetry_summary.csv")


if __name__ == "__main__":
    main()
