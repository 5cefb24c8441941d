"""Host-side trace generation reproduces the reference's generate_requests()."""

from __future__ import annotations

import json

import numpy as np
import pytest

import paper_2601_04250_b200 as gg
from tests import _golden as G


@pytest.mark.parametrize("name", ["closed_k2", "poisson_k4", "onoff_k4", "closed_k1000"])
def test_trace_matches_reference(name):
    d = G.npz("workload_" + name)
    cfg = json.loads(str(d["config"]))
    wl = gg.WorkloadConfig(mode=gg.ArrivalMode[cfg["mode"]], rate_rps=cfg["rate_rps"],
                           on_rate_rps=cfg["on_rate_rps"], off_rate_rps=cfg["off_rate_rps"],
                           phase_mean_s=cfg["phase_mean_s"], num_requests=cfg["num_requests"],
                           num_classes=cfg["num_classes"], confidence_low=cfg["confidence_low"],
                           confidence_high=cfg["confidence_high"])
    rng = np.random.default_rng(np.random.SeedSequence(cfg["seed"]).spawn(3)[0])
    tr = gg.generate_trace(wl, cfg["horizon_s"], rng)
    assert np.array_equal(tr.arrival_t, d["arrival_t"], equal_nan=True)
    assert np.array_equal(tr.scores, d["scores"])
    assert np.array_equal(tr.true_label, d["true_label"])
    # the generator ends in the same state as the reference's (one variate past the horizon)
    rng2 = np.random.default_rng(np.random.SeedSequence(cfg["seed"]).spawn(3)[0])
    reqs = gg.generate_requests(wl, cfg["horizon_s"], rng2)
    assert rng.random() == rng2.random()
    assert [r.top_class() for r in reqs] == list(tr.top_class)


def test_workload_validation():
    with pytest.raises(gg.ConfigError):
        gg.WorkloadConfig(num_classes=1)
    with pytest.raises(gg.ConfigError):
        gg.WorkloadConfig(num_classes=4, confidence_low=0.2)
    with pytest.raises(gg.ConfigError):
        gg.WorkloadConfig(mode=gg.ArrivalMode.POISSON, rate_rps=0.0)
