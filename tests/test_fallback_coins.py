"""The fallback coin stream drawn on the host == the reference simulator's
`_fb_rng` draws (servesim.py:177-180, 254), so the device accounting consumes
the same coins.  CPU test; skipped when the reference package is absent."""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _greengate():
    for p in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(p, "greengate")):
            if p not in sys.path:
                sys.path.insert(0, p)
            import greengate
            return greengate
    pytest.skip("reference package not available")


@pytest.mark.parametrize("seed", [0, 11, 42])
def test_fallback_coins_match_reference_stream(seed):
    gg_ref = _greengate()
    from paper_2601_04250_b200.serving import fallback_coins
    sim = gg_ref.Simulation(gg_ref.SimConfig(seed=seed))
    want = np.array([float(sim._fb_rng.random()) for _ in range(257)])
    assert np.array_equal(fallback_coins(seed, 257), want)
