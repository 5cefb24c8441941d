"""Parity of the device controller (K1/K2/K3 through the C ABI) with the oracle.

Decisions must match bit-exactly except requests with |J - tau| < EPS_BAND
(north star; none occur in these fixtures).  Utility/J/tau values must match
within MAX_ULP ulps (CUDA's fp64 log/exp vs glibc's are both ~0.5-1 ulp);
their exact-match rate is recorded.  Integer work (codes, counts, admitted
index lists, window order) is compared exactly.
"""

from __future__ import annotations

import math

import numpy as np
import pytest

from oracle import c_oracle
from oracle import controller_oracle as O
from tests import _golden as G

pytestmark = pytest.mark.gpu

EPS_BAND = 1e-12
MAX_ULP = 4


def ulp_diff(a, b) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float64).view(np.int64)
    b = np.ascontiguousarray(b, dtype=np.float64).view(np.int64)
    a = np.where(a < 0, np.int64(-0x8000000000000000) - a, a)
    b = np.where(b < 0, np.int64(-0x8000000000000000) - b, b)
    return np.abs(a - b)


def assert_close_ulp(got, want, what):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    both_nan = np.isnan(got) & np.isnan(want)
    d = np.where(both_nan, 0, ulp_diff(got, want))
    assert d.max(initial=0) <= MAX_ULP, f"{what}: max ulp {d.max()}"
    return int((d != 0).sum())


@pytest.fixture(scope="module")
def gg():
    import paper_2601_04250_b200 as gg
    return gg


@pytest.fixture(scope="module")
def torch():
    import torch
    return torch


def test_library_is_native(gg):
    from paper_2601_04250_b200 import _native
    lib = _native.load()
    assert b"sm_100a" in lib.gg_version()


def test_literal_kats(gg):
    kat = G.kat()
    for scores, ent, omc in kat["utility_literal"]:
        assert abs(gg.entropy_utility(scores) - ent) <= 2 * math.ulp(max(ent, 1e-300)) or \
            gg.entropy_utility(scores) == ent
        assert gg.one_minus_confidence_utility(scores) == omc
    # exact goldens the reference's tests pin (test_gateway.py:52, test_controller.py:95)
    assert gg.entropy_utility([0.5, 0.5]) == 1.0
    assert gg.entropy_utility([1.0, 0.0]) == 0.0
    assert abs(gg.entropy_utility([0.9, 0.1]) - 0.46899559358928117) <= 1e-12
    for bad in ([1.0], [0.7, 0.7], [0.5, 0.6], [-0.1, 1.1], [0.5, math.nan]):
        with pytest.raises(gg.InvalidDistribution):
            gg.entropy_utility(bad)
        with pytest.raises(gg.InvalidDistribution):
            gg.one_minus_confidence_utility(bad)
    got = [gg.threshold_at(gg.ThresholdSchedule(a, b, k, t0), t)
           for a, b, k, t0, t, _ in kat["threshold_at"][:300]]
    want = [w for *_, w in kat["threshold_at"][:300]]
    assert_close_ulp(got, want, "threshold_at")
    assert gg.threshold_at(gg.ThresholdSchedule(1.0, 0.2, 0.5), 0.0) == 1.0
    for a, b, g, u, e, c, want in kat["cost"][:100]:
        assert gg.cost(gg.CostWeights(a, b, g), u, e, c) == want


def test_decide_literal(gg):
    for (tau, scores, direction, proxy, beta, admit, path, u, e, c, j, th) in G.kat()["decide_literal"]:
        cfg = gg.ControllerConfig(alpha=1.0, beta=beta, gamma=0.0, tau0=tau, tau_inf=tau, k=1.0,
                                  direction=[gg.Direction.GEQ, gg.Direction.LT][direction],
                                  utility_proxy=[gg.UtilityProxy.ENTROPY,
                                                 gg.UtilityProxy.ONE_MINUS_CONFIDENCE][proxy])
        ctl = cfg.build(gg.EnergyLedger())
        d = ctl.decide(gg.RequestFeatures(0, 0.0, tuple(scores)), now=0.0)
        assert d.admit == admit
        assert d.path.name == ["NONE", "DIRECT", "BATCHED"][path]
        b = d.breakdown
        assert (b.energy, b.congestion, b.threshold) == (e, c, th)
        assert_close_ulp([b.utility, b.composite], [u, j], "decide literal")
    ctl = gg.ControllerConfig(tau0=0.5, tau_inf=0.5, k=1.0).build(gg.EnergyLedger())
    ctl.decide(gg.RequestFeatures(0, 0.0, (0.5, 0.5)), 0.0)
    ctl.decide(gg.RequestFeatures(0, 0.0, (0.99, 0.01)), 0.0)
    assert (ctl.admitted_total, ctl.skipped_total) == (1, 1)
    with pytest.raises(gg.InvalidDistribution):
        ctl.decide(gg.RequestFeatures(0, 0.0, (0.7, 0.7)), 0.0)
    assert (ctl.admitted_total, ctl.skipped_total) == (1, 1)


def test_outcome_literals(gg):
    ctl = gg.ControllerConfig(tau0=0.5, tau_inf=0.5, k=1.0).build(gg.EnergyLedger())
    ctl.record_outcome(10.0, 2.0, 0)
    assert ctl.ledger.ewma_joules_per_request == 2.0
    ctl.record_outcome(10.0, 4.0, 0)
    assert ctl.ledger.ewma_joules_per_request == 0.9 * 2.0 + (1.0 - 0.9) * 4.0
    with pytest.raises(gg.NegativeMeasurement):
        ctl.record_outcome(-1.0, 1.0, 0)
    ctl2 = gg.ControllerConfig().build(gg.EnergyLedger())
    for lat in range(1, 101):
        ctl2.record_outcome(float(lat), 1.0, 0)
    assert ctl2.p95_ms() == 95.0            # test_controller.py:262-266
    ctl2.reset_clock(10.0)
    assert gg.threshold_at(ctl2.schedule, 10.0) == 1.0


@pytest.mark.parametrize("k", [2, 3, 4, 10, 100, 1000])
def test_utility_rows(gg, torch, k):
    from paper_2601_04250_b200 import _native
    d = G.npz("dist_rows")
    rows, ent, omc, valid = d[f"rows_k{k}"], d[f"entropy_k{k}"], d[f"omc_k{k}"], d[f"valid_k{k}"]
    lib = _native.load()
    x = torch.from_numpy(rows).cuda()
    n = rows.shape[0]
    for proxy, want in ((0, ent), (1, omc)):
        u = torch.empty(n, dtype=torch.float64, device="cuda")
        v = torch.empty(n, dtype=torch.uint8, device="cuda")
        _native.check("gg_utility", lib.gg_utility(_native.ptr(x), n, k, k, proxy, _native.ptr(u),
                                                   _native.ptr(v), _native.stream_ptr()))
        assert np.array_equal(v.cpu().numpy().astype(bool), valid)
        mism = assert_close_ulp(u.cpu().numpy()[valid], want[valid], f"utility k={k} proxy={proxy}")
        if proxy == 1:
            assert mism == 0
        print(f"k={k} proxy={proxy}: {mism}/{valid.sum()} rows differ in the last bits")


def _snap(gg, d, i):
    return gg.CongestionSnapshot(int(d["snap_qd"][i]), float(d["snap_p95"][i]), float(d["snap_fill"][i]))


@pytest.mark.parametrize("name", G.SIM_NAMES)
def test_sim_capture_through_public_api(gg, name):
    """Replay a full reference simulation's controller calls through the drop-in."""
    d = G.sim(name)
    p = d["params"]
    current = {"snap": None}
    cfg = gg.ControllerConfig(alpha=p["alpha"], beta=p["beta"], gamma=p["gamma"], tau0=p["tau0"],
                              tau_inf=p["tau_inf"], k=p["k"],
                              direction=[gg.Direction.GEQ, gg.Direction.LT][p["direction"]],
                              utility_proxy=[gg.UtilityProxy.ENTROPY,
                                             gg.UtilityProxy.ONE_MINUS_CONFIDENCE][p["utility_proxy"]],
                              routing=list(gg.RoutePolicy)[p["routing"]],
                              queue_threshold=p["queue_threshold"])
    ctl = cfg.build(gg.EnergyLedger(ewma_lambda=p["ewma_lambda"]), lambda: current["snap"],
                    p95_window=p["p95_window"])
    codes, u, e, c, j, tau = [], [], [], [], [], []
    idx = []
    for i in range(len(d["kind"])):
        if d["kind"][i] == 0:
            current["snap"] = _snap(gg, d, i)
            dec = ctl.decide(gg.RequestFeatures(i, float(d["now"][i]),
                                                tuple(float(x) for x in d["scores"][i])),
                             float(d["now"][i]))
            codes.append({"NONE": 0, "DIRECT": 1, "BATCHED": 2}[dec.path.name])
            b = dec.breakdown
            u.append(b.utility); e.append(b.energy); c.append(b.congestion)
            j.append(b.composite); tau.append(b.threshold)
            idx.append(i)
        else:
            ctl.record_outcome(float(d["lat"][i]), float(d["joules"][i]), int(d["qd"][i]))
    idx = np.array(idx)
    codes = np.array(codes)
    want_j, want_tau = d["j"][idx], d["tau"][idx]
    band = np.abs(want_j - want_tau) < EPS_BAND
    assert np.array_equal(codes[~band], d["code"][idx][~band])
    assert band.sum() == 0
    assert np.array_equal(np.array(e), d["e"][idx]) and np.array_equal(np.array(c), d["c"][idx])
    for arr, key in ((u, "u"), (j, "j"), (tau, "tau")):
        assert_close_ulp(arr, d[key][idx], f"{name}:{key}")
    st = G.state_dict_of_abi(ctl.state_struct())
    want = dict(d["final_state"])
    st.pop("total_joules"), want.pop("total_joules")
    assert st == want


@pytest.mark.parametrize("name", G.REPLAY_NAMES)
def test_replay_batch_api(gg, torch, name):
    """Micro-batched replay: decide_batch per step (frozen snapshot) + record_outcomes."""
    d = G.replay(name)
    p = d["params"]
    cfg = gg.ControllerConfig(alpha=p["alpha"], beta=p["beta"], gamma=p["gamma"], tau0=p["tau0"],
                              tau_inf=p["tau_inf"], k=p["k"],
                              direction=[gg.Direction.GEQ, gg.Direction.LT][p["direction"]],
                              utility_proxy=[gg.UtilityProxy.ENTROPY,
                                             gg.UtilityProxy.ONE_MINUS_CONFIDENCE][p["utility_proxy"]],
                              routing=list(gg.RoutePolicy)[p["routing"]],
                              queue_threshold=p["queue_threshold"])
    ctl = cfg.build(gg.EnergyLedger(ewma_lambda=p["ewma_lambda"]), p95_window=p["p95_window"])
    rows = torch.from_numpy(d["rows"]).cuda()
    now = torch.from_numpy(d["now"]).cuda()
    B = int(d["batch"])
    n = rows.shape[0]
    got_codes = np.empty(n, np.uint8)
    got_bd = np.empty((n, 3))
    for s, s0 in enumerate(range(0, n, B)):
        snap = gg.CongestionSnapshot(int(d["step_qd"][s]), float(d["step_p95"][s]),
                                     float(d["step_fill"][s]))
        out = ctl.decide_batch(rows[s0:s0 + B], now[s0:s0 + B], snap)
        dec = out.decision.cpu().numpy()
        got_codes[s0:s0 + B] = dec
        got_bd[s0:s0 + B] = out.breakdown.cpu().numpy()
        summ = out.summary()
        adm = np.nonzero((dec == 1) | (dec == 2))[0]
        assert np.array_equal(out.admitted_idx[: summ["n_admitted"]].cpu().numpy(), adm)
        if summ["n_invalid"] < len(dec):
            assert (summ["energy"], summ["congestion"]) == (d["e_step"][s], d["c_step"][s])
        m = d["out_step"] == s
        if m.any():
            ctl.record_outcomes(torch.from_numpy(d["out_lat"][m]).cuda(),
                                torch.from_numpy(d["out_joules"][m]).cuda(),
                                torch.from_numpy(d["out_qd"][m]).cuda())
    band = np.abs(d["j"] - d["tau"]) < EPS_BAND
    assert np.array_equal(got_codes[~band], d["code"][~band])
    for col, key in enumerate(("u", "j", "tau")):
        mism = assert_close_ulp(got_bd[:, col], d[key], f"{name}:{key}")
        print(f"{name}:{key}: {mism}/{n} differ in last bits")
    st = G.state_dict_of_abi(ctl.state_struct())
    assert st == d["final_state"]


@pytest.mark.parametrize("n,k", [(0, 2), (1, 2), (1023, 2), (1025, 4), (4_194_304, 2),
                                 (100_003, 4), (3000, 7), (2048, 1000), (129, 37),
                                 (1_500_007, 4), (1_300_001, 5)])   # the last two: split path
@pytest.mark.parametrize("breakdown", [True, False])
def test_admit_vs_c_oracle_large(gg, torch, n, k, breakdown):
    """Order-preserving compaction and counters at scale vs the C oracle."""
    rng = np.random.default_rng(n + k)
    if k == 2:
        c = rng.uniform(0.5, 1.0, size=n)
        rows = np.stack([c, 1.0 - c], axis=1)
    else:
        base = rng.integers(1, 50, size=(n, k))
        rows = G.rows_from_base(base)
    if n > 10:
        rows[7] = np.nan            # invalid rows
        rows[n // 2, 0] = -0.25
    now = np.sort(rng.uniform(0.0, 10.0, size=n))
    p = dict(alpha=1.0, beta=0.3, gamma=0.2, tau0=0.9, tau_inf=0.3, k=0.7, ewma_lambda=0.9,
             direction=0, utility_proxy=0, routing=2, queue_threshold=3, p95_window=100)
    orc = c_oracle.COracle(G.abi_params(p))
    orc.outcome(np.array([3.0, 5.0, 4.0]), np.array([1.0, 2.0, 1.5]), np.array([1, 5, 2]))
    snap = (4, 5.0, 0.25)
    dec_o, bd_o, idx_o, info_o = orc.admit(rows, now, snap)
    cfg = gg.ControllerConfig(alpha=1.0, beta=0.3, gamma=0.2, tau0=0.9, tau_inf=0.3, k=0.7,
                              routing=gg.RoutePolicy.THRESHOLD_ON_QUEUE, queue_threshold=3)
    ctl = cfg.build(gg.EnergyLedger())
    ctl.record_outcomes(torch.tensor([3.0, 5.0, 4.0], dtype=torch.float64, device="cuda"),
                        torch.tensor([1.0, 2.0, 1.5], dtype=torch.float64, device="cuda"),
                        torch.tensor([1, 5, 2], dtype=torch.int32, device="cuda"))
    # with a breakdown: the exact path; without: the fast filter + exact refinement
    out = ctl.decide_batch(torch.from_numpy(rows).cuda(), torch.from_numpy(now).cuda(),
                           gg.CongestionSnapshot(*snap), breakdown=breakdown)
    dec = out.decision.cpu().numpy()
    band = np.abs(bd_o[:, 1] - bd_o[:, 2]) < EPS_BAND
    assert np.array_equal(dec[~band], dec_o[~band])
    summ = out.summary()
    assert summ["n_invalid"] == info_o.n_invalid
    assert summ["first_invalid"] == info_o.first_invalid
    assert summ["n_admitted"] == info_o.n_admitted
    assert np.array_equal(out.admitted_idx[: summ["n_admitted"]].cpu().numpy(), idx_o)
    if breakdown:
        assert_close_ulp(out.breakdown.cpu().numpy(), bd_o, f"admit n={n} k={k}")
    st = G.state_dict_of_abi(ctl.state_struct())
    assert st == G.state_dict_of_abi(orc.state)


@pytest.mark.parametrize("n,k", [(4096, 2), (4096, 4), (4096, 1000), (1_250_000, 2)])
def test_fast_filter_near_threshold(gg, torch, n, k):
    """Rows engineered to sit within the fast-path margin of tau take the exact
    path; decisions must still equal the oracle's bit-for-bit."""
    rng = np.random.default_rng(k)
    base = rng.integers(1, 60, size=(n, k))
    rows = G.rows_from_base(base)
    p = dict(alpha=1.0, beta=0.0, gamma=0.0, tau0=0.5, tau_inf=0.5, k=1.0, ewma_lambda=0.9,
             direction=0, utility_proxy=0, routing=0, queue_threshold=4, p95_window=100)
    orc0 = c_oracle.COracle(G.abi_params(p))
    _d, bd0, _i, _f = orc0.admit(rows, np.zeros(n))
    tau = float(np.median(bd0[:, 0]))          # threshold inside the utility distribution
    p.update(tau0=tau, tau_inf=tau)
    orc = c_oracle.COracle(G.abi_params(p))
    dec_o, bd_o, idx_o, info_o = orc.admit(rows, np.zeros(n))
    # tau is the median utility, so some rows sit inside the fast filter's margin
    assert np.min(np.abs(bd_o[:, 0] - tau)) < 1e-3
    ctl = gg.ControllerConfig(tau0=tau, tau_inf=tau, k=1.0).build(gg.EnergyLedger())
    out = ctl.decide_batch(torch.from_numpy(rows).cuda(), torch.zeros(n, dtype=torch.float64,
                                                                      device="cuda"),
                           breakdown=False)
    band = np.abs(bd_o[:, 1] - bd_o[:, 2]) < EPS_BAND
    assert np.array_equal(out.decision.cpu().numpy()[~band], dec_o[~band])
    assert np.array_equal(out.admitted_idx[: out.n_admitted].cpu().numpy(), idx_o)


def test_epilogue_vs_oracle(gg, torch):
    from paper_2601_04250_b200 import _native
    lib = _native.load()
    rng = np.random.default_rng(5)
    for n, k in ((64, 1000), (128, 2), (3, 4)):
        logits = (rng.standard_normal((n, k)) * 4).astype(np.float32)
        logits[0, 1] = logits[0].max()        # tie: first max wins
        x = torch.from_numpy(logits).cuda()
        probs = torch.empty((n, k), dtype=torch.float64, device="cuda")
        am = torch.empty(n, dtype=torch.int32, device="cuda")
        conf = torch.empty(n, dtype=torch.float64, device="cuda")
        util = torch.empty(n, dtype=torch.float64, device="cuda")
        _native.check("gg_epilogue", lib.gg_epilogue(
            _native.ptr(x), n, k, k, 0, _native.ptr(probs), _native.ptr(am), _native.ptr(conf),
            _native.ptr(util), _native.stream_ptr()))
        p_o, am_o = c_oracle.softmax(logits)
        p = probs.cpu().numpy()
        assert np.allclose(p, p_o, rtol=1e-13, atol=1e-300)
        assert np.array_equal(am.cpu().numpy(), am_o)
        assert np.array_equal(conf.cpu().numpy(), p.max(axis=1))
        for i in range(n):   # every row passes the reference's validation
            xs = [float(v) for v in p[i]]
            assert abs(O.neumaier_sum(xs) - 1.0) <= 1e-9
            assert util.cpu().numpy()[i] == O.entropy_utility(xs) or \
                abs(util.cpu().numpy()[i] - O.entropy_utility(xs)) <= 4 * math.ulp(1.0)
