"""Pin the CPU oracle (oracle/) to the reference before trusting it.

Every check compares the Python restatement (oracle/controller_oracle.py) and
the C restatement (oracle/gg_oracle.c) with values produced by the reference
implementation itself (tests/golden/, made by make_golden.py from
/root/reference/pkg/src): the literal known-answer cases of the reference's
own tests, seeded random cases, full-simulation event logs and micro-batched
replays.  Equality is bit-exact (==) throughout.
"""

from __future__ import annotations

import math
import random

import numpy as np
import pytest

from oracle import c_oracle
from oracle import controller_oracle as O
from tests import _golden as G

KAT = G.kat()


def _same(a: float, b: float) -> bool:
    return (a == b) or (math.isnan(a) and math.isnan(b))


# ------------------------------------------------------------------ sum / KATs

def test_neumaier_matches_cpython_sum():
    rng = random.Random(3)
    for _ in range(3000):
        k = rng.randint(1, 60)
        xs = [rng.random() * 10 ** rng.randint(-8, 8) * rng.choice((1, -1)) for _ in range(k)]
        assert O.neumaier_sum(xs) == sum(xs)
    assert O.neumaier_sum([0.1] * 10) == 1.0


def test_threshold_kat():
    for tau0, tinf, k, t0, t, want in KAT["threshold_at"]:
        assert O.threshold_at(tau0, tinf, k, t0, t) == want


def test_reference_literal_threshold_values():
    # pkg/tests/test_controller.py:41-56
    assert O.threshold_at(1.0, 0.2, 0.5, 0.0, 0.0) == 1.0
    assert abs(O.threshold_at(1.0, 0.2, 0.5, 0.0, 2.0) - 0.4943035529371539) <= 1e-12
    assert O.threshold_at(1.0, 0.2, 0.5, 100.0, 50.0) == 1.0


def test_utility_kat():
    for scores, ent, omc in KAT["utility_literal"]:
        assert O.entropy_utility(scores) == ent
        assert O.one_minus_confidence_utility(scores) == omc
    assert O.entropy_utility([0.5, 0.5]) == 1.0          # test_gateway.py:52
    assert abs(O.entropy_utility([0.9, 0.1]) - 0.46899559358928117) <= 1e-12


def test_invalid_distributions_kat():
    for text, rejected in KAT["utility_invalid"]:
        scores = eval(text, {"nan": math.nan, "inf": math.inf})  # repr of a float list
        if rejected:
            with pytest.raises(O.OracleInvalidDistribution):
                O.entropy_utility(scores)
        else:
            O.entropy_utility(scores)


def test_cost_kat():
    for a, b, g, u, e, c, want in KAT["cost"]:
        assert O.cost(a, b, g, u, e, c) == want


def test_normalizer_kat():
    for ops in KAT["normalizer"]:
        ch = O.Channel()
        for op, raw, want in ops:
            if op == "observe":
                ch.observe(raw)
            else:
                assert ch.normalize(raw) == want


def test_ewma_kat():
    for lam, xs, vals in KAT["ewma"]:
        prev = None
        for x, want in zip(xs, vals):
            prev = O.ewma_update(prev, x, lam)
            assert prev == want


def test_p95_kat():
    for values, want in KAT["p95"]:
        assert O.percentile_nearest_rank(values, 95.0) == want


def test_decide_literal_kat():
    for (tau, scores, direction, proxy, beta, admit, path, u, e, c, j, th) in KAT["decide_literal"]:
        ctl = O.OracleController(O.OracleParams(beta=beta, tau0=tau, tau_inf=tau, k=1.0,
                                                direction=direction, utility_proxy=proxy))
        d = ctl.decide(scores, 0.0)
        assert (d.admit, d.code) == (admit, path)
        assert (d.utility, d.energy, d.congestion, d.composite, d.threshold) == (u, e, c, j, th)


@pytest.mark.parametrize("k", [2, 3, 4, 10, 100, 1000])
def test_distribution_rows(k):
    d = G.npz("dist_rows")
    rows, ent, omc, valid = d[f"rows_k{k}"], d[f"entropy_k{k}"], d[f"omc_k{k}"], d[f"valid_k{k}"]
    for i in range(rows.shape[0]):
        xs = [float(x) for x in rows[i]]
        if not valid[i]:
            with pytest.raises(O.OracleInvalidDistribution):
                O.entropy_utility(xs)
            continue
        assert O.entropy_utility(xs) == ent[i]
        assert O.one_minus_confidence_utility(xs) == omc[i]
    # the C restatement, entropy and 1-conf proxies
    for proxy, want in ((O.ENTROPY, ent), (O.ONE_MINUS_CONFIDENCE, omc)):
        p = G.abi_params(dict(alpha=1.0, beta=0.0, gamma=0.0, tau0=0.5, tau_inf=0.5, k=1.0,
                              ewma_lambda=0.9, direction=0, utility_proxy=proxy, routing=0,
                              queue_threshold=4, p95_window=100))
        orc = c_oracle.COracle(p)
        dec, bd, _idx, _info = orc.admit(rows, np.zeros(rows.shape[0]))
        assert np.array_equal(dec == 255, ~valid)
        assert np.array_equal(bd[valid, 0], want[valid])


# ------------------------------------------------------- full-simulation captures

@pytest.mark.parametrize("name", G.SIM_NAMES)
def test_sim_capture_python_oracle(name):
    d = G.sim(name)
    ctl = O.OracleController(O.OracleParams(**d["params"]))
    nd = 0
    for i in range(len(d["kind"])):
        if d["kind"][i] == 0:
            snap = (int(d["snap_qd"][i]), float(d["snap_p95"][i]), float(d["snap_fill"][i]))
            got = ctl.decide([float(x) for x in d["scores"][i]], float(d["now"][i]), snap)
            want = (int(d["code"][i]), d["u"][i], d["e"][i], d["c"][i], d["j"][i], d["tau"][i])
            assert (got.code, got.utility, got.energy, got.congestion, got.composite,
                    got.threshold) == want, (name, i)
            nd += 1
        else:
            ctl.record_outcome(float(d["lat"][i]), float(d["joules"][i]), int(d["qd"][i]))
    want = {k: tuple(v) if isinstance(v, list) else v for k, v in d["final_state"].items()}
    got = ctl.state_tuple()
    # the simulator's ledger also books baseline draw at the end (servesim.py:389)
    want.pop("total_joules"), got.pop("total_joules")
    assert got == want
    assert ctl.admitted_total == int(d["admitted"])
    assert nd == int(d["admitted"]) + int(d["skipped"])


@pytest.mark.parametrize("name", G.SIM_NAMES)
def test_sim_capture_c_oracle(name):
    d = G.sim(name)
    orc = c_oracle.COracle(G.abi_params(d["params"]))
    for i in range(len(d["kind"])):
        if d["kind"][i] == 0:
            snap = (int(d["snap_qd"][i]), float(d["snap_p95"][i]), float(d["snap_fill"][i]))
            dec, bd, _idx, info = orc.admit(d["scores"][i:i + 1], d["now"][i:i + 1], snap)
            assert dec[0] == d["code"][i], (name, i)
            assert (bd[0, 0], bd[0, 1], bd[0, 2]) == (d["u"][i], d["j"][i], d["tau"][i])
            assert (info.energy, info.congestion) == (d["e"][i], d["c"][i])
        else:
            assert orc.outcome(d["lat"][i:i + 1], d["joules"][i:i + 1], d["qd"][i:i + 1]) == -1
    got, want = G.state_dict_of_abi(orc.state), dict(d["final_state"])
    got.pop("total_joules"), want.pop("total_joules")  # baseline draw, servesim.py:389
    assert got == want


# ------------------------------------------------------------ micro-batched replays

def run_replay_c(d: dict):
    orc = c_oracle.COracle(G.abi_params(d["params"]))
    B = int(d["batch"])
    n = d["rows"].shape[0]
    for s, s0 in enumerate(range(0, n, B)):
        snap = (int(d["step_qd"][s]), float(d["step_p95"][s]), float(d["step_fill"][s]))
        dec, bd, idx, info = orc.admit(d["rows"][s0:s0 + B], d["now"][s0:s0 + B], snap)
        yield s, s0, dec, bd, idx, info
        m = d["out_step"] == s
        assert orc.outcome(d["out_lat"][m], d["out_joules"][m], d["out_qd"][m]) == -1
    assert G.state_dict_of_abi(orc.state) == d["final_state"]


@pytest.mark.parametrize("name", G.REPLAY_NAMES)
def test_replay_c_oracle(name):
    d = G.replay(name)
    B = int(d["batch"])
    for s, s0, dec, bd, idx, info in run_replay_c(d):
        sl = slice(s0, s0 + B)
        assert np.array_equal(dec, d["code"][sl])
        for col, key in enumerate(("u", "j", "tau")):
            assert np.array_equal(bd[:, col], d[key][sl], equal_nan=True)
        assert np.array_equal(idx, np.nonzero((dec == 1) | (dec == 2))[0])
        if info.n_invalid < len(dec):
            assert (info.energy, info.congestion) == (d["e_step"][s], d["c_step"][s])


def test_replay_python_oracle_k2():
    d = G.replay("k2_ablation")
    ctl = O.OracleController(O.OracleParams(**d["params"]))
    B = int(d["batch"])
    n = d["rows"].shape[0]
    for s, s0 in enumerate(range(0, n, B)):
        snap = (int(d["step_qd"][s]), float(d["step_p95"][s]), float(d["step_fill"][s]))
        rows = [[float(x) for x in r] for r in d["rows"][s0:s0 + B]]
        out = ctl.decide_batch(rows, [float(x) for x in d["now"][s0:s0 + B]], snap)
        assert [o.code for o in out] == list(d["code"][s0:s0 + B])
        for lat, jo, q in zip(d["out_lat"][d["out_step"] == s], d["out_joules"][d["out_step"] == s],
                              d["out_qd"][d["out_step"] == s]):
            ctl.record_outcome(float(lat), float(jo), int(q))
    assert ctl.ewma == d["final_state"]["ewma"]
    assert ctl.p95_ms() == d["final_state"]["p95_current"]
