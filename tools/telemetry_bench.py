"""CPU timing of the columnar JSONL export vs the reference's per-record
dict + json.dumps loop, same bytes, N records (default 1M).  Not a GPU number.

    python tools/telemetry_bench.py [n]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2601_04250_b200.telemetry import JSONL_FIELDS, jsonl_bytes  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
    rng = np.random.default_rng(0)
    enq = np.cumsum(rng.exponential(0.01, n))
    cols = dict(request_id=np.arange(n), admitted=rng.random(n) < 0.5,
                path=np.array(["DIRECT", "BATCHED", "NONE"])[rng.integers(0, 3, n)],
                enqueue_t=enq, start_t=enq + 0.001, finish_t=enq + 0.02, latency_ms=rng.random(n) * 30,
                joules=rng.random(n) * 5, predicted_label=rng.integers(0, 1000, n), correct=rng.random(n) < 0.5)
    t0 = time.perf_counter()
    ours = jsonl_bytes(*(cols[f] for f in JSONL_FIELDS))
    t1 = time.perf_counter()
    lists = [cols[f].tolist() for f in JSONL_FIELDS]
    ref = "".join(json.dumps(dict(zip(JSONL_FIELDS, rec))) + "\n" for rec in zip(*lists))
    t2 = time.perf_counter()
    assert ours == ref
    print(f"{n} records: columnar {t1 - t0:.2f} s, per-record json.dumps {t2 - t1:.2f} s "
          f"({(t2 - t1) / (t1 - t0):.1f}x), {len(ours) / 1e6:.0f} MB, identical bytes")


if __name__ == "__main__":
    main()
