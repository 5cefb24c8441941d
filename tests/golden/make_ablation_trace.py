"""Golden JSONL trace of the reference's ablation run, written BY the reference.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_ablation_trace.py

Runs `greengate.run(ablation_reference())` (presets.py, 100 closed-loop
requests, 58 admitted) with the unmodified reference and writes its
`export_jsonl` bytes to tests/golden/ablation_trace.jsonl.
tests/test_reference_suite_gpu.py compares the patched (device-controller)
run's bytes with this file.
"""

import os
import sys

import greengate
from greengate.presets import ablation_reference

out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ablation_trace.jsonl")
trace = greengate.run(ablation_reference())
assert trace.admitted == 58
greengate.export_jsonl(trace, out)
print(f"wrote {out} ({trace.arrivals} records, python {sys.version.split()[0]})")
