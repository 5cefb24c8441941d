"""Generate golden fixtures from the REFERENCE implementation (build container only).

Run here, where the read-only reference exists:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports `greengate` from /root/reference/pkg/src, runs the reference's own
code, and writes small fixtures next to this script.  Nothing at test, smoke or
bench time reads /root/reference; the fixtures travel with the repo.

Fixtures
  kat.json               known-answer values of the reference functions: the
                         literal cases of pkg/tests/test_controller.py,
                         test_energy.py, test_telemetry.py, test_gateway.py plus
                         seeded random cases (threshold_at, entropy_utility,
                         one_minus_confidence_utility, cost, normalizers, EWMA,
                         nearest-rank p95).
  dist_rows.npz          random distributions K in {2,3,4,10,100,1000} and the
                         reference's entropy / 1-conf of every row.
  sim_<name>.npz         event logs of full reference simulations (servesim.run)
                         captured at the controller boundary: every decide()
                         with the snapshot the congestion source returned and the
                         reference AdmissionDecision, every record_outcome()
                         with its arguments, plus the final controller state.
  replay_<name>.npz      micro-batched replays through the reference's public
                         API: per step `decide` x B against one frozen snapshot,
                         then `record_outcome` for each admitted row in order.
  workload_<name>.npz    reference generate_requests() output (arrival times,
                         scores, labels) for seeds/configs the package's trace
                         generator must reproduce.
"""

from __future__ import annotations

import json
import math
import os
import sys
from dataclasses import replace

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.dont_write_bytecode = True
sys.path.insert(0, REF)

import greengate  # noqa: E402
from greengate import controller as gc  # noqa: E402
from greengate import energy as ge  # noqa: E402
from greengate import servesim as gs  # noqa: E402
from greengate import telemetry as gt  # noqa: E402
from greengate import workload as gw  # noqa: E402
from greengate import presets as gp  # noqa: E402

DIR = {gc.Direction.GEQ: 0, gc.Direction.LT: 1}
UTIL = {gc.UtilityProxy.ENTROPY: 0, gc.UtilityProxy.ONE_MINUS_CONFIDENCE: 1}
ROUTE = {gc.RoutePolicy.ALL_DIRECT: 0, gc.RoutePolicy.ALL_BATCHED: 1,
         gc.RoutePolicy.THRESHOLD_ON_QUEUE: 2}
PATH = {gc.ServicePath.NONE: 0, gc.ServicePath.DIRECT: 1, gc.ServicePath.BATCHED: 2}


def params_of(cc: gc.ControllerConfig, ewma_lambda: float, p95_window: int) -> dict:
    return dict(alpha=cc.alpha, beta=cc.beta, gamma=cc.gamma, tau0=cc.tau0,
                tau_inf=cc.tau_inf, k=cc.k, ewma_lambda=ewma_lambda,
                direction=DIR[cc.direction], utility_proxy=UTIL[cc.utility_proxy],
                routing=ROUTE[cc.routing], queue_threshold=cc.queue_threshold,
                p95_window=p95_window)


def state_of(ctl: gc.AdmissionController) -> dict:
    def ch(c):
        return None if c.running_min is None else [c.running_min, c.running_max]
    n = ctl.normalizers
    return dict(energy=ch(n.energy), queue_depth=ch(n.queue_depth), p95_ms=ch(n.p95_ms),
                ewma=ctl.ledger.ewma_joules_per_request,
                samples_seen=ctl.ledger.samples_seen,
                total_joules=ctl.ledger.total_joules,
                admitted_total=ctl.admitted_total, skipped_total=ctl.skipped_total,
                p95_current=ctl.p95_ms(), t_origin=ctl.schedule.t_origin)


# --------------------------------------------------------------------------- KATs

def make_kat() -> dict:
    kat: dict = {"python": sys.version, "reference": "greengate " + greengate.__version__}
    # threshold_at: test_controller.py:41-78 literal cases + random triples.
    th = []
    for (tau0, tinf, k, t0, t) in [(1.0, 0.2, 0.5, 0.0, 0.0), (1.0, 0.2, 0.5, 0.0, 1e6),
                                   (1.0, 0.2, 0.5, 0.0, 2.0), (1.0, 0.2, 0.5, 100.0, 50.0),
                                   (1.0, 0.2, 0.5, 100.0, 100.0), (0.4, 0.4, 2.0, 0.0, 5.0),
                                   (0.9, 0.35, 2.0, 0.0, 0.25), (1.0, 0.2, 1.0, 10.0, 10.0)]:
        th.append([tau0, tinf, k, t0, t, gc.threshold_at(gc.ThresholdSchedule(tau0, tinf, k, t0), t)])
    rng = np.random.default_rng(2024)
    for _ in range(2000):
        tinf = float(rng.uniform(0.0, 1.0))
        tau0 = tinf + float(rng.uniform(0.0, 2.0))
        k = float(rng.uniform(0.01, 8.0))
        t0 = float(rng.uniform(-5.0, 5.0))
        t = float(rng.uniform(-10.0, 60.0))
        th.append([tau0, tinf, k, t0, t, gc.threshold_at(gc.ThresholdSchedule(tau0, tinf, k, t0), t)])
    kat["threshold_at"] = th

    # utilities: literal cases of test_controller.py:94-128, test_gateway.py:47-64
    lit = [[0.5, 0.5], [1.0, 0.0], [0.9, 0.1], [0.25, 0.25, 0.25, 0.25],
           [0.26, 0.25, 0.25, 0.24], [0.0, 1.0, 0.0], [0.001, 0.999], [0.99, 0.01],
           [0.8, 0.2], [0.6, 0.4], [0.1] * 10, [0.7, 0.1, 0.1, 0.1]]
    kat["utility_literal"] = [[s, gc.entropy_utility(s), gc.one_minus_confidence_utility(s)] for s in lit]
    bad = [[1.0], [0.7, 0.7], [0.5, 0.6], [-0.1, 1.1], [0.5, math.nan], [0.5, math.inf],
           [1.0 + 2e-9, 0.0], [1.0 + 5e-10, 0.0], [0.5, 0.5 - 1.5e-9]]
    ok_bad = []
    for s in bad:
        try:
            gc.entropy_utility(s)
            ok_bad.append([repr(s), False])
        except gc.InvalidDistribution:
            ok_bad.append([repr(s), True])
    kat["utility_invalid"] = ok_bad

    # cost: test_controller.py:156-172
    cost_cases = [[0.0, 0.0, 0.0, 0.3, 0.9, 0.1], [1.0, 1.0, 1.0, 0.5, 0.2, 0.3],
                  [0.5, 0.3, 0.2, 0.468995, 0.25, 0.1]]
    rng = np.random.default_rng(99)
    for _ in range(500):
        cost_cases.append([float(x) for x in rng.uniform(-1.0, 1.0, size=3)]
                          + [float(x) for x in rng.uniform(0.0, 1.0, size=3)])
    kat["cost"] = [c + [gc.cost(gc.CostWeights(*c[:3]), *c[3:])] for c in cost_cases]

    # normalizer: test_controller.py:133-151 + random observe/normalize sequences
    seqs = []
    rng = np.random.default_rng(5)
    for _ in range(200):
        chan = gc.NormalizerChannel()
        ops = []
        for _ in range(int(rng.integers(1, 12))):
            raw = float(rng.choice([rng.uniform(-5, 5), float(rng.integers(0, 4))]))
            if rng.random() < 0.4:
                chan.observe(raw)
                ops.append(["observe", raw, None])
            else:
                ops.append(["normalize", raw, chan.normalize(raw)])
        seqs.append(ops)
    kat["normalizer"] = seqs

    # EWMA: test_energy.py:16-35, test_controller.py:237-249
    ew = []
    rng = np.random.default_rng(8)
    for _ in range(300):
        lam = float(rng.uniform(0.01, 0.99))
        prev = None
        xs = [float(x) for x in rng.exponential(3.0, size=int(rng.integers(1, 20)))]
        vals = []
        for x in xs:
            prev = ge.ewma_update(prev, x, lam)
            vals.append(prev)
        ew.append([lam, xs, vals])
    kat["ewma"] = ew

    # percentile_nearest_rank: test_telemetry.py:48-75 (incl. 1..100 -> 95)
    pc = [[list(map(float, range(1, 101))), gt.percentile_nearest_rank(list(map(float, range(1, 101))), 95.0)]]
    rng = np.random.default_rng(6)
    for _ in range(300):
        v = [float(x) for x in rng.normal(10.0, 4.0, size=int(rng.integers(1, 200)))]
        pc.append([v, gt.percentile_nearest_rank(v, 95.0)])
    kat["p95"] = pc

    # decision literals: test_controller.py:182-228
    def one(tau, scores, direction=gc.Direction.GEQ, proxy=gc.UtilityProxy.ENTROPY, beta=0.0):
        ctl = gc.ControllerConfig(alpha=1.0, beta=beta, gamma=0.0, tau0=tau, tau_inf=tau, k=1.0,
                                  direction=direction, utility_proxy=proxy).build(ge.EnergyLedger())
        d = ctl.decide(gw.RequestFeatures(0, 0.0, tuple(scores), None), now=0.0)
        b = d.breakdown
        return [tau, scores, DIR[direction], UTIL[proxy], beta, d.admit, PATH[d.path],
                b.utility, b.energy, b.congestion, b.composite, b.threshold]
    kat["decide_literal"] = [
        one(0.5, [0.5, 0.5]), one(0.5, [0.99, 0.01]), one(0.5, [0.5, 0.5], gc.Direction.LT),
        one(0.5, [0.99, 0.01], gc.Direction.LT), one(1.0, [0.5, 0.5]), one(0.0, [0.5, 0.5], beta=1.0),
        one(0.5, [0.9, 0.1]), one(0.05, [0.9, 0.1], proxy=gc.UtilityProxy.ONE_MINUS_CONFIDENCE),
        one(0.9, [0.5, 0.5]), one(0.9, [1.0, 0.0])]
    return kat


# ------------------------------------------------------------------ distributions

def make_dist_rows() -> dict:
    rng = np.random.default_rng(77)
    out = {}
    for k, n in [(2, 4000), (3, 2000), (4, 2000), (10, 1000), (100, 300), (1000, 200)]:
        raw = rng.exponential(1.0, size=(n, k))
        if k >= 10:  # peaked rows, like a classifier's softmax
            raw = raw ** 4
        rows = raw / raw.sum(axis=1, keepdims=True)
        if k == 2:  # the synthetic K=2 scores are (c, 1-c)
            c = rng.uniform(0.5, 1.0, size=n)
            rows[: n // 2, 0] = c[: n // 2]
            rows[: n // 2, 1] = 1.0 - c[: n // 2]
        rows[0, :] = 0.0
        rows[0, 0] = 1.0
        if k == 2:
            rows[1] = [0.5, 0.5]
        ent = np.empty(n)
        omc = np.empty(n)
        valid = np.ones(n, dtype=bool)
        for i in range(n):
            xs = [float(x) for x in rows[i]]
            try:
                ent[i] = gc.entropy_utility(xs)
                omc[i] = gc.one_minus_confidence_utility(xs)
            except gc.InvalidDistribution:
                valid[i] = False
                ent[i] = omc[i] = np.nan
        out[f"rows_k{k}"] = rows
        out[f"entropy_k{k}"] = ent
        out[f"omc_k{k}"] = omc
        out[f"valid_k{k}"] = valid
    return out


# -------------------------------------------------------------- simulation capture

def capture_sim(config: gs.SimConfig) -> dict:
    """Run the reference simulator, logging every controller call in order."""
    kinds, nows, scores, sqd, sp95, sfill = [], [], [], [], [], []
    lat, jou, oqd = [], [], []
    ou, oe, oc, oj, otau, ocode = [], [], [], [], [], []

    class Capture(gs.Simulation):
        def __init__(self, cfg):
            super().__init__(cfg)
            ctl = self.controller
            src = ctl.congestion_source
            last = {}

            def source():
                snap = src()
                last["snap"] = snap
                return snap
            ctl.congestion_source = source
            real_decide, real_outcome = ctl.decide, ctl.record_outcome

            def decide(features, now):
                d = real_decide(features, now)
                s = last["snap"]
                kinds.append(0); nows.append(now); scores.append(list(features.scores))
                sqd.append(s.queue_depth); sp95.append(s.p95_latency_ms); sfill.append(s.batch_fill)
                lat.append(0.0); jou.append(0.0); oqd.append(0)
                b = d.breakdown
                ou.append(b.utility); oe.append(b.energy); oc.append(b.congestion)
                oj.append(b.composite); otau.append(b.threshold); ocode.append(PATH[d.path])
                return d

            def outcome(latency_ms, joules, queue_depth):
                real_outcome(latency_ms, joules, queue_depth)
                kinds.append(1); nows.append(0.0); scores.append(None)
                sqd.append(0); sp95.append(0.0); sfill.append(0.0)
                lat.append(latency_ms); jou.append(joules); oqd.append(queue_depth)
                for arr in (ou, oe, oc, oj, otau):
                    arr.append(0.0)
                ocode.append(0)
            ctl.decide, ctl.record_outcome = decide, outcome

    sim = Capture(config)
    trace = sim.run()
    k = config.workload.num_classes
    sc = np.zeros((len(kinds), k))
    for i, s in enumerate(scores):
        if s is not None:
            sc[i] = s
    cc = config.controller
    return dict(
        params=json.dumps(params_of(cc, config.ewma_lambda, config.p95_window)),
        final_state=json.dumps(state_of(sim.controller)),
        kind=np.array(kinds, np.int8), now=np.array(nows), scores=sc,
        snap_qd=np.array(sqd, np.int64), snap_p95=np.array(sp95), snap_fill=np.array(sfill),
        lat=np.array(lat), joules=np.array(jou), qd=np.array(oqd, np.int32),
        u=np.array(ou), e=np.array(oe), c=np.array(oc), j=np.array(oj), tau=np.array(otau),
        code=np.array(ocode, np.uint8),
        admitted=np.int64(trace.admitted), skipped=np.int64(trace.skipped),
    )


def demo03(horizon=25.0, **cc) -> gs.SimConfig:
    """pkg/demos/03_dual_path_simulation.py:26-42 with a longer horizon."""
    base = dict(tau0=0.9, tau_inf=0.35, k=2.0, routing=gc.RoutePolicy.THRESHOLD_ON_QUEUE,
                queue_threshold=2)
    base.update(cc)
    return gs.SimConfig(
        seed=11, horizon_s=horizon, concurrency=2, baseline_power_w=50.0,
        path_a=gs.PathAConfig(latency_mean_ms=5.0, latency_std_ms=1.2, active_energy_j_per_req=2.5),
        path_b=gs.PathBConfig(max_batch_size=8, batching_window_ms=10.0, batch_base_ms=4.0,
                              per_item_ms=1.0, batch_base_energy_j=6.0, per_item_energy_j=1.5),
        controller=gc.ControllerConfig(**base),
        workload=gw.WorkloadConfig(mode=gw.ArrivalMode.POISSON, rate_rps=400.0, num_classes=4,
                                   confidence_low=0.55, confidence_high=0.97))


def sim_configs() -> dict:
    sweep = gp.energy_sweep_reference()
    onoff = replace(demo03(beta=-0.3, gamma=0.4), workload=gw.WorkloadConfig(
        mode=gw.ArrivalMode.ONOFF, on_rate_rps=800.0, off_rate_rps=50.0, phase_mean_s=0.5,
        num_classes=4, confidence_low=0.55, confidence_high=0.97))
    return {
        "demo03": demo03(),
        "demo03_all_channels": demo03(beta=-0.3, gamma=0.4),
        "ablation": gp.ablation_reference(),
        "energy_sweep": replace(sweep, horizon_s=50.0,
                                controller=replace(sweep.controller, beta=0.5)),
        "onoff_bursty": onoff,
        "lt_omc": demo03(horizon=10.0, direction=gc.Direction.LT,
                         utility_proxy=gc.UtilityProxy.ONE_MINUS_CONFIDENCE,
                         tau0=0.2, tau_inf=0.05, beta=0.2, gamma=-0.5),
    }


# --------------------------------------------------------------- micro-batched replay

def replay(name: str, rows: np.ndarray, nows: np.ndarray, cc: gc.ControllerConfig,
           batch: int, seed: int, p95_window: int = 100, ewma_lambda: float = 0.9) -> dict:
    """Drive the reference public API as the GPU loop does."""
    snap = {"v": gs.CongestionSnapshot(0, 0.0, 0.0)}
    ctl = cc.build(ge.EnergyLedger(ewma_lambda=ewma_lambda), lambda: snap["v"],
                   p95_window=p95_window)
    rng = np.random.default_rng(seed)
    n = rows.shape[0]
    codes = np.zeros(n, np.uint8)
    u = np.zeros(n); j = np.zeros(n); tau = np.zeros(n)
    step_qd, step_p95, step_fill = [], [], []
    out_lat, out_j, out_qd, out_step = [], [], [], []
    e_step, c_step, states = [], [], []
    pending = 0
    for s0 in range(0, n, batch):
        qd = int(pending)
        s = gs.CongestionSnapshot(qd, ctl.p95_ms(), min(1.0, pending / 64.0))
        snap["v"] = s
        step_qd.append(s.queue_depth); step_p95.append(s.p95_latency_ms); step_fill.append(s.batch_fill)
        adm = []
        e_here = c_here = 0.0
        for i in range(s0, min(n, s0 + batch)):
            try:
                d = ctl.decide(gw.RequestFeatures(i, float(nows[i]), tuple(float(x) for x in rows[i]), None),
                               float(nows[i]))
            except gc.InvalidDistribution:
                codes[i] = 255
                u[i] = j[i] = tau[i] = np.nan
                continue
            codes[i] = PATH[d.path]
            b = d.breakdown
            u[i], j[i], tau[i] = b.utility, b.composite, b.threshold
            e_here, c_here = b.energy, b.congestion
            if d.admit:
                adm.append(i)
        e_step.append(e_here); c_step.append(c_here)
        nadm = len(adm)
        for r, _i in enumerate(adm):
            lat_ms = 2.0 + 0.25 * nadm + float(rng.exponential(0.5))
            joules = 1.5 + 6.0 / max(1, nadm) + float(rng.uniform(0.0, 0.2))
            depth = int(rng.integers(0, 12))
            ctl.record_outcome(lat_ms, joules, depth)
            out_lat.append(lat_ms); out_j.append(joules); out_qd.append(depth)
            out_step.append(s0 // batch)
        pending = int(rng.integers(0, 80))
        states.append([ctl.ledger.ewma_joules_per_request, ctl.p95_ms(), ctl.admitted_total,
                       ctl.skipped_total])
    return dict(
        params=json.dumps(params_of(cc, ewma_lambda, p95_window)), batch=np.int64(batch),
        rows=rows, now=nows, code=codes, u=u, j=j, tau=tau,
        step_qd=np.array(step_qd, np.int64), step_p95=np.array(step_p95),
        step_fill=np.array(step_fill), e_step=np.array(e_step), c_step=np.array(c_step),
        out_lat=np.array(out_lat), out_joules=np.array(out_j), out_qd=np.array(out_qd, np.int32),
        out_step=np.array(out_step, np.int64), step_state=np.array(states),
        final_state=json.dumps(state_of(ctl)),
    )


def rows_from_base(base: np.ndarray) -> np.ndarray:
    """Exact, platform-independent rows: integer fourth powers over their integer sum.

    Also used by tests (tests/golden/__init__ helpers) to rebuild the rows; row 5
    gets one negative entry (an invalid distribution) in the K=1000 replay.
    """
    num = base.astype(np.int64) ** 4
    den = num.sum(axis=1, keepdims=True)
    rows = num.astype(np.float64) / den.astype(np.float64)
    return rows


def make_replays() -> dict:
    out = {}
    # K=2 ablation workload (presets.py:64-96) at 20,480 requests, B=128
    wl = replace(gp.ablation_reference().workload, num_requests=20_480)
    reqs = gw.generate_requests(wl, 10.0, np.random.default_rng(np.random.SeedSequence(42).spawn(3)[0]))
    rows = np.array([r.scores for r in reqs])
    nows = np.arange(len(reqs)) * 0.0005
    cc = gc.ControllerConfig(alpha=1.0, beta=-0.3, gamma=0.4, tau0=0.9, tau_inf=0.39796077431433013,
                             k=0.5, routing=gc.RoutePolicy.THRESHOLD_ON_QUEUE, queue_threshold=40)
    out["k2_ablation"] = replay("k2_ablation", rows, nows, cc, batch=128, seed=1)
    # K=1000 peaked random rows (ResNet-like), B=64.  Rows are rebuilt exactly
    # from small integers (rows_from_base below) so the fixture stores 2 B/entry.
    rng = np.random.default_rng(1000)
    base = rng.integers(1, 1200, size=(1024, 1000)).astype(np.uint16)
    rows = rows_from_base(base)
    rows[5, 3] = -1e-3  # one invalid row
    nows = np.arange(1024) * 0.002
    cc = gc.ControllerConfig(alpha=1.0, beta=0.25, gamma=0.3, tau0=1.0, tau_inf=0.55, k=1.5,
                             routing=gc.RoutePolicy.ALL_BATCHED)
    d = replay("k1000_softmax", rows, nows, cc, batch=64, seed=2)
    d["rows_base"] = base
    d["patch"] = np.array([5.0, 3.0, -1e-3])  # rows[5, 3] = -1e-3 after rows_from_base
    del d["rows"]
    out["k1000_softmax"] = d
    # K=4 demo-03 scores, one_minus_confidence + LT
    wl = gw.WorkloadConfig(mode=gw.ArrivalMode.CLOSED, num_requests=8192, num_classes=4,
                           confidence_low=0.55, confidence_high=0.97)
    reqs = gw.generate_requests(wl, 1.0, np.random.default_rng(3))
    rows = np.array([r.scores for r in reqs])
    nows = np.arange(len(reqs)) * 0.001
    cc = gc.ControllerConfig(alpha=1.0, beta=0.1, gamma=0.2, tau0=0.1, tau_inf=0.3, k=0.8,
                             direction=gc.Direction.LT,
                             utility_proxy=gc.UtilityProxy.ONE_MINUS_CONFIDENCE)
    out["k4_lt_omc"] = replay("k4_lt_omc", rows, nows, cc, batch=256, seed=3, p95_window=37)
    return out


# ------------------------------------------------------------------------ workloads

def make_workloads() -> dict:
    out = {}
    cases = {
        "closed_k2": (replace(gp.ablation_reference().workload, num_requests=3000), 10.0, 42),
        "poisson_k4": (sim_configs()["demo03"].workload, 5.0, 11),
        "onoff_k4": (sim_configs()["onoff_bursty"].workload, 5.0, 11),
        "closed_k1000": (gw.WorkloadConfig(mode=gw.ArrivalMode.CLOSED, num_requests=300,
                                           num_classes=1000, confidence_low=0.3,
                                           confidence_high=0.9), 1.0, 7),
    }
    for name, (wl, horizon, seed) in cases.items():
        rng = np.random.default_rng(np.random.SeedSequence(seed).spawn(3)[0])
        reqs = gw.generate_requests(wl, horizon, rng)
        out[name] = dict(
            config=json.dumps(dict(mode=wl.mode.value, rate_rps=wl.rate_rps,
                                   on_rate_rps=wl.on_rate_rps, off_rate_rps=wl.off_rate_rps,
                                   phase_mean_s=wl.phase_mean_s, num_requests=wl.num_requests,
                                   num_classes=wl.num_classes, confidence_low=wl.confidence_low,
                                   confidence_high=wl.confidence_high, horizon_s=horizon,
                                   seed=seed)),
            arrival_t=np.array([r.arrival_t for r in reqs]),
            scores=np.array([r.scores for r in reqs]),
            true_label=np.array([r.true_label for r in reqs], np.int64),
        )
    return out


def main() -> None:
    with open(os.path.join(HERE, "kat.json"), "w") as f:
        json.dump(make_kat(), f)
    np.savez_compressed(os.path.join(HERE, "dist_rows.npz"), **make_dist_rows())
    for name, cfg in sim_configs().items():
        np.savez_compressed(os.path.join(HERE, f"sim_{name}.npz"), **capture_sim(cfg))
    for name, d in make_replays().items():
        np.savez_compressed(os.path.join(HERE, f"replay_{name}.npz"), **d)
    for name, d in make_workloads().items():
        np.savez_compressed(os.path.join(HERE, f"workload_{name}.npz"), **d)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
