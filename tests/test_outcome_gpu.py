"""K2 (gg_outcome) vs the C oracle for every register-window instantiation.

record_outcome() sequences with random latencies (ties included), window
capacities 1 .. 1024 (1, 2, 4, 8, 16, 32 register slots per lane), checked
after every chunk: EWMA, sample count, window contents in arrival order,
nearest-rank p95 and normalizer channels — all bit-exact.
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import c_oracle
from tests import _golden as G

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("window", [1, 5, 32, 33, 100, 200, 500, 1000, 1024])
def test_outcome_windows(window):
    import torch
    import paper_2601_04250_b200 as gg
    rng = np.random.default_rng(window)
    p = dict(alpha=1.0, beta=0.0, gamma=0.0, tau0=0.5, tau_inf=0.5, k=1.0, ewma_lambda=0.8,
             direction=0, utility_proxy=0, routing=0, queue_threshold=4, p95_window=window)
    orc = c_oracle.COracle(G.abi_params(p))
    ctl = gg.ControllerConfig(tau0=0.5, tau_inf=0.5, k=1.0).build(
        gg.EnergyLedger(ewma_lambda=0.8), p95_window=window)
    for chunk in range(6):
        n = int(rng.integers(1, 700))
        lat = np.round(rng.exponential(5.0, size=n), 1)   # rounding makes ties common
        jo = rng.uniform(0.0, 3.0, size=n)
        qd = rng.integers(0, 20, size=n).astype(np.int32)
        orc.outcome(lat, jo, qd)
        ctl.record_outcomes(torch.from_numpy(lat).cuda(), torch.from_numpy(jo).cuda(),
                            torch.from_numpy(qd).cuda())
        s = ctl.state_struct()
        o = orc.state
        assert G.state_dict_of_abi(s) == G.state_dict_of_abi(o), (window, chunk)
        cnt = s.win_count
        assert cnt == o.win_count and s.win_head == o.win_head
        assert list(s.win)[:window] == list(o.win)[:window]
        assert list(s.win_sorted)[:cnt] == sorted(list(o.win)[:cnt])
