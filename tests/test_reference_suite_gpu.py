"""Drop-in proof at the reference's own call sites (VERDICT r1 "next" #8).

The unmodified reference package is installed offline into baseline/_ref by
tools/install_reference.sh (with its test suite, demos and configs under
baseline/_ref/greengate_suite/).  With `patch_greengate` applied, every
`ControllerConfig.build` the reference makes — the simulator
(servesim.py:185-190), the HTTP gateway (gateway.py:51-56), the tests' own
`config.build(EnergyLedger())` — returns the sm_100a controller, and:

* the reference's own test suite passes against it (subprocess, plugin
  tools/greengate_patch_plugin.py; the plugin's report proves the device
  controller served the decisions);
* `greengate.run(ablation_reference())` admits 58/100 (tests/test_servesim.py:91-97)
  and its JSONL trace is byte-identical to the unpatched reference run's and to
  the golden the reference wrote here (tests/golden/ablation_trace.jsonl);
* a demo-03 style 10k-request run (THRESHOLD_ON_QUEUE, all three channels)
  makes the same decisions as the unpatched reference.

Skipped when baseline/_ref is absent (nothing here reads /root/reference).
"""

from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
SUITE = os.path.join(REF, "greengate_suite")
GOLDEN = os.path.join(ROOT, "tests", "golden")


@pytest.fixture(scope="module")
def greengate():
    if not os.path.isdir(os.path.join(REF, "greengate")):
        pytest.skip("reference not installed (tools/install_reference.sh)")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import greengate as gg_ref
    return gg_ref


def _run(gg_ref, cfg, patched: bool):
    from paper_2601_04250_b200.integration import patch_greengate, unpatch_greengate
    if patched:
        patch_greengate(gg_ref)
    try:
        return gg_ref.run(cfg)
    finally:
        unpatch_greengate(gg_ref)


def _jsonl(gg_ref, trace, tmp_path, name):
    p = tmp_path / name
    gg_ref.export_jsonl(trace, str(p))
    return p.read_bytes()


def test_ablation_reference_through_patch(greengate, tmp_path):
    from greengate.presets import ablation_reference
    from paper_2601_04250_b200.controller import AdmissionController
    t_dev = _run(greengate, ablation_reference(), patched=True)
    t_ref = _run(greengate, ablation_reference(), patched=False)
    assert t_dev.admitted == 58 and t_ref.admitted == 58
    assert t_dev.makespan_s == pytest.approx(58 * 0.005, abs=1e-9)
    b_dev = _jsonl(greengate, t_dev, tmp_path, "dev.jsonl")
    assert b_dev == _jsonl(greengate, t_ref, tmp_path, "ref.jsonl")
    with open(os.path.join(GOLDEN, "ablation_trace.jsonl"), "rb") as f:
        assert b_dev == f.read()
    # the patched simulator really held the device controller
    sim = greengate.Simulation.__new__(greengate.Simulation)
    from paper_2601_04250_b200.integration import patch_greengate, unpatch_greengate
    patch_greengate(greengate)
    try:
        sim.__init__(ablation_reference())
        assert isinstance(sim.controller, AdmissionController)
    finally:
        unpatch_greengate(greengate)


def test_demo03_all_channels_through_patch(greengate):
    """10,000 Poisson arrivals, THRESHOLD_ON_QUEUE, beta/gamma != 0: the device
    controller's decisions, paths and ledger equal the reference's."""
    from dataclasses import replace
    from greengate import (ArrivalMode, ControllerConfig, PathAConfig, PathBConfig, RoutePolicy,
                           SimConfig, WorkloadConfig)
    cfg = SimConfig(seed=11, horizon_s=25.0, concurrency=4,
                    path_a=PathAConfig(latency_mean_ms=8.0, latency_std_ms=2.0,
                                       active_energy_j_per_req=3.0),
                    path_b=PathBConfig(max_batch_size=8, batching_window_ms=10.0, batch_base_ms=6.0,
                                       per_item_ms=1.5, batch_base_energy_j=8.0,
                                       per_item_energy_j=1.0),
                    controller=ControllerConfig(alpha=1.0, beta=-0.3, gamma=0.4, tau0=0.9,
                                                tau_inf=0.35, k=2.0,
                                                routing=RoutePolicy.THRESHOLD_ON_QUEUE,
                                                queue_threshold=2),
                    workload=WorkloadConfig(mode=ArrivalMode.POISSON, rate_rps=400.0,
                                            num_classes=4, confidence_low=0.55,
                                            confidence_high=0.97))
    t_dev = _run(greengate, cfg, patched=True)
    t_ref = _run(greengate, cfg, patched=False)
    assert t_ref.arrivals == 10000
    assert t_dev.admitted == t_ref.admitted and t_dev.skipped == t_ref.skipped
    assert [(r.request_id, r.admitted, r.path) for r in t_dev.records] == \
        [(r.request_id, r.admitted, r.path) for r in t_ref.records]
    assert t_dev.ledger.ewma_joules_per_request == t_ref.ledger.ewma_joules_per_request
    assert t_dev.ledger.samples_seen == t_ref.ledger.samples_seen
    del replace


def test_reference_test_suite_with_device_controller(greengate, tmp_path):
    """The reference's own tests (controller, simulator, gateway over HTTP,
    acceptance criteria, CLI) run with every ControllerConfig.build patched to
    the device controller."""
    if not os.path.isdir(os.path.join(SUITE, "tests")):
        pytest.skip("reference suite not copied (tools/install_reference.sh)")
    report = tmp_path / "patch_report.json"
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([REF, ROOT, os.path.join(ROOT, "tools")]),
               GG_PATCH_REPORT=str(report), PYTHONDONTWRITEBYTECODE="1")
    tests = [os.path.join(SUITE, "tests", f) for f in
             ("test_controller.py", "test_servesim.py", "test_gateway.py", "test_acceptance.py",
              "test_energy.py", "test_telemetry.py", "test_workload.py", "test_presets.py",
              "test_config.py", "test_cli.py")]
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider",
                        "-p", "greengate_patch_plugin", *tests],
                       cwd=SUITE, env=env, capture_output=True, text=True, timeout=1200)
    tail = "\n".join((r.stdout + r.stderr).splitlines()[-30:])
    print(tail)
    assert r.returncode == 0, tail
    rep = json.loads(report.read_text())
    assert rep["greengate"].startswith(REF)
    assert rep["device_controllers"] > 50 and rep["decide_calls"] > 10000, rep
