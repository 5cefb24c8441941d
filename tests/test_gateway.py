"""Gateway micro-batching front end (paper_2601_04250_b200.gateway).

The reference gateway applies one controller call per request under a lock
(gateway.py:179-230).  `GatewayBatcher` must give every request the answer the
sequential gateway gives for the same request order, while coalescing runs of
decides into one K1 launch and runs of outcomes into one K2 launch.

CPU tests: the batcher's host logic (ordering, run splitting at depth / score
count changes, 400 / 422 errors, depth updates) against the oracle-backed
sequential gateway, with an oracle-backed stand-in controller.  GPU test: the
real controller through the C ABI against the same sequential oracle gateway.
"""

from __future__ import annotations

import math
import random
from types import SimpleNamespace

import pytest

from oracle import controller_oracle as O

PARAMS = dict(alpha=1.0, beta=-0.1, gamma=-0.3, tau0=0.9, tau_inf=0.3, k=0.05, ewma_lambda=0.9,
              routing=O.THRESHOLD_ON_QUEUE, queue_threshold=4)


def _requests(seed=7, n=300):
    """A mixed stream: decides (k = 3, some k = 2, some invalid, some with depth),
    outcomes (some negative), in one total order."""
    rng = random.Random(seed)
    reqs = []
    t = 1.0
    for i in range(n):
        t += rng.random() * 0.5
        r = rng.random()
        if r < 0.7:
            k = 3 if rng.random() < 0.85 else 2
            xs = [rng.random() for _ in range(k)]
            s = sum(xs)
            xs = [x / s for x in xs]
            if rng.random() < 0.04:
                xs[0] += 0.5                        # does not sum to 1 -> 400
            body = {"id": f"r{i}", "scores": xs, "timestamp_s": t}
            if rng.random() < 0.15:
                body["queue_depth"] = rng.randrange(0, 9)
            reqs.append(("decide", body))
        else:
            lat = rng.random() * 40.0
            if rng.random() < 0.05:
                lat = -1.0                          # negative -> 400, no state change
            reqs.append(("outcome", {"id": f"o{i}", "latency_ms": lat, "joules": rng.random() * 5.0,
                                     "queue_depth": rng.randrange(0, 9)}))
    return reqs


def sequential_gateway(reqs):
    """The reference gateway's handlers over the oracle, one request at a time."""
    ctl = O.OracleController(O.OracleParams(**PARAMS), t_origin=0.0)
    depth = 0
    out = []
    for kind, b in reqs:
        if kind == "reset":
            ctl.reset_clock(b["t_origin"])
            out.append(None)
            continue
        if kind == "decide":
            if "queue_depth" in b:
                depth = b["queue_depth"]
            try:
                d = ctl.decide(b["scores"], float(b["timestamp_s"]), (depth, ctl.p95_ms(), 0.0))
            except O.OracleInvalidDistribution:
                out.append(400)
                continue
            out.append({"admit": d.admit, "path": {O.SKIP: "NONE", O.DIRECT: "DIRECT", O.BATCHED: "BATCHED"}[d.code],
                        "j": d.composite, "tau": d.threshold, "l": d.utility, "e": d.energy,
                        "c": d.congestion, "reason": "ADMITTED" if d.admit else "BELOW_THRESHOLD"})
        else:
            try:
                ctl.record_outcome(b["latency_ms"], b["joules"], b["queue_depth"])
            except O.OracleNegativeMeasurement:
                out.append(400)
                continue
            depth = b["queue_depth"]
            out.append(None)
    return out, ctl


class OracleBackedController:
    """Stand-in for AdmissionController on CPU: decide_batch / record_outcomes over the oracle."""

    def __init__(self):
        import torch
        from paper_2601_04250_b200.controller import Direction
        self.o = O.OracleController(O.OracleParams(**PARAMS), t_origin=0.0)
        self.device = torch.device("cpu")
        self.direction = Direction.GEQ
        self.calls = []

    def p95_ms(self):
        return self.o.p95_ms()

    def decide_batch(self, scores, now, snap, breakdown=True):
        import torch
        from paper_2601_04250_b200 import _abi
        self.calls.append(("decide", int(scores.shape[0])))
        res = self.o.decide_batch(scores.tolist(), now.tolist(),
                                  (snap.queue_depth, snap.p95_latency_ms, snap.batch_fill))
        ok = [r for r in res if r is not None]
        info = _abi.gg_batch_info()
        if ok:
            info.energy, info.congestion = ok[-1].energy, ok[-1].congestion
        return SimpleNamespace(
            decision=torch.tensor([255 if r is None else r.code for r in res], dtype=torch.uint8),
            breakdown=torch.tensor([[0.0] * 3 if r is None else [r.utility, r.composite, r.threshold]
                                    for r in res], dtype=torch.float64),
            info=torch.frombuffer(bytearray(bytes(info)), dtype=torch.uint8))

    def record_outcomes(self, lat, jl, qd, check=True):
        self.calls.append(("outcome", int(lat.shape[0])))
        for a, b, c in zip(lat.tolist(), jl.tolist(), qd.tolist()):
            self.o.record_outcome(a, b, c)

    def reset_clock(self, t):
        self.o.reset_clock(t)


def _run_batched(gw, reqs):
    sub = {"decide": gw.submit_decide, "outcome": gw.submit_outcome,
           "reset": lambda b: gw.submit_reset()}
    futs = [sub[kind](b) for kind, b in reqs]
    out = []
    for f in futs:
        try:
            out.append(f.result(timeout=60))
        except Exception as exc:   # ApiError
            out.append(getattr(exc, "status", exc))
    return out


def _expected_runs(reqs):
    """Launch counts the run splitting must produce when everything is drained at once."""
    dec = outc = 0
    depth, prev = 0, None
    for kind, b in reqs:
        if kind == "decide":
            if "queue_depth" in b:
                depth = b["queue_depth"]
            key = ("d", len(b["scores"]), depth)
            if key != prev:
                dec += 1
            prev = key
        else:
            if prev is None or prev[0] != "o":
                outc += 1
            if b["latency_ms"] >= 0:
                depth = b["queue_depth"]
            prev = ("o",)
    return dec, outc


def test_batcher_matches_sequential_gateway_cpu():
    from paper_2601_04250_b200.gateway import GatewayBatcher
    reqs = _requests()
    want, octl = sequential_gateway(reqs)
    fake = OracleBackedController()
    # max_batch = the whole stream and a long wait: one deterministic drain
    with GatewayBatcher(None, controller=fake, max_batch=len(reqs), max_wait_s=30.0, clock=lambda: 0.0) as gw:
        got = _run_batched(gw, reqs)
    assert got == want
    dec, outc = _expected_runs(reqs)
    assert sum(1 for c in fake.calls if c[0] == "decide") == dec
    assert sum(1 for c in fake.calls if c[0] == "outcome") <= outc   # all-negative runs launch nothing
    assert dec < sum(1 for k, _ in reqs if k == "decide") / 2        # it did batch
    assert fake.o.state_tuple() == octl.state_tuple()


def test_batcher_field_errors_cpu():
    from paper_2601_04250_b200.gateway import ApiError, GatewayBatcher
    with GatewayBatcher(None, controller=OracleBackedController(), max_wait_s=0.0) as gw:
        for body, status in [({"scores": [0.5, 0.5]}, 422), ({"id": "a"}, 422),
                             ({"id": "a", "scores": [0.5, True]}, 422),
                             ({"id": "a", "scores": [0.5, 0.5], "queue_depth": 1.5}, 422),
                             ({"id": 3, "scores": [0.5, 0.5]}, 422)]:
            with pytest.raises(ApiError) as e:
                gw.decide(body)
            assert e.value.status == status
        with pytest.raises(ApiError) as e:
            gw.decide({"id": "a", "scores": [1.0], "timestamp_s": 1.0})
        assert e.value.status == 400
        with pytest.raises(ApiError) as e:
            gw.outcome({"id": "a", "latency_ms": 1.0, "joules": -1.0, "queue_depth": 0})
        assert e.value.status == 400
        r = gw.decide({"id": "a", "scores": [0.5, 0.5], "timestamp_s": 1.0})
        assert r["l"] == 1.0 and r["reason"] in ("ADMITTED", "BELOW_THRESHOLD")
    with GatewayBatcher(None) as gw:
        with pytest.raises(ApiError) as e:
            gw.decide({"id": "a", "scores": [0.5, 0.5]})
        assert e.value.status == 503


def _ulp(a, b):
    import numpy as np
    a, b = np.float64(a).view(np.int64), np.float64(b).view(np.int64)
    return abs(int(a) - int(b))


@pytest.mark.gpu
def test_batcher_device_controller_vs_sequential_oracle():
    """The real K1 / K2 launches behind the batcher vs the sequential oracle gateway:
    decisions, paths, reasons and errors exact; j / tau / l / e / c within 4 ulp."""
    import paper_2601_04250_b200 as gg
    from paper_2601_04250_b200.gateway import GatewayBatcher
    reqs = _requests(seed=11, n=400)
    want, _ = sequential_gateway(reqs)
    cfg = gg.ControllerConfig(alpha=PARAMS["alpha"], beta=PARAMS["beta"], gamma=PARAMS["gamma"],
                              tau0=PARAMS["tau0"], tau_inf=PARAMS["tau_inf"], k=PARAMS["k"],
                              routing=gg.RoutePolicy.THRESHOLD_ON_QUEUE,
                              queue_threshold=PARAMS["queue_threshold"])
    with GatewayBatcher(cfg, clock=lambda: 0.0, max_batch=len(reqs), max_wait_s=30.0) as gw:
        got = _run_batched(gw, reqs)
        assert gw.launches["decide"] == _expected_runs(reqs)[0]   # one K1 launch per run
    assert len(got) == len(want)
    for g, w in zip(got, want):
        if not isinstance(w, dict):
            assert g == w
            continue
        for key in ("admit", "path", "reason"):
            assert g[key] == w[key]
        for key in ("j", "tau", "l", "e", "c"):
            assert _ulp(g[key], w[key]) <= 4 or (math.isnan(g[key]) and math.isnan(w[key])), key


def test_batcher_concurrent_clients_cpu():
    """8 client threads hammer decide/outcome concurrently: every answer equals the
    sequential gateway's answer for the enqueue order the batcher recorded, and the
    final controller state matches."""
    import threading
    from paper_2601_04250_b200.gateway import GatewayBatcher
    reqs = _requests(seed=23, n=800)
    per = [reqs[i::8] for i in range(8)]
    fake = OracleBackedController()
    answers = {}
    with GatewayBatcher(None, controller=fake, max_wait_s=50e-6, clock=lambda: 0.0,
                        record_order=True) as gw:
        def client(part):
            for kind, b in part:
                try:
                    r = gw.decide(b) if kind == "decide" else gw.outcome(b)
                except Exception as exc:
                    r = getattr(exc, "status", exc)
                answers[b["id"]] = r
        ts = [threading.Thread(target=client, args=(p,)) for p in per]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        order = list(gw.order)
    assert len(order) == len(reqs)
    want, octl = sequential_gateway(order)
    for (kind, b), w in zip(order, want):
        assert answers[b["id"]] == w, (kind, b["id"])
    assert fake.o.state_tuple() == octl.state_tuple()
    assert len(fake.calls) < len(reqs)   # requests were coalesced


def test_batcher_reset_in_request_order_cpu():
    """POST /v1/reset is applied by the worker in enqueue order: decides queued
    before it see the old clock origin, decides after it the new one; the
    recorded order replays through the sequential gateway; a closed gateway
    answers 503 instead of blocking."""
    import itertools
    from paper_2601_04250_b200.gateway import ApiError, GatewayBatcher
    reqs = _requests(seed=5, n=200)
    reqs = reqs[:60] + [("reset", {})] + reqs[60:140] + [("reset", {})] + reqs[140:]
    ticks = itertools.count(1)
    fake = OracleBackedController()
    with GatewayBatcher(None, controller=fake, max_batch=len(reqs), max_wait_s=30.0,
                        clock=lambda: 0.5 * next(ticks), record_order=True) as gw:
        got = _run_batched(gw, reqs)
        order = list(gw.order)
    want, octl = sequential_gateway(order)
    assert [k for k, _ in order].count("reset") == 2
    assert got == want
    assert fake.o.state_tuple() == octl.state_tuple()
    for call in (gw.flush, gw.reset, lambda: gw.decide({"id": "a", "scores": [0.5, 0.5]}),
                 lambda: gw.outcome({"id": "a", "latency_ms": 1.0, "joules": 1.0, "queue_depth": 0})):
        with pytest.raises(ApiError) as e:
            call()
        assert e.value.status == 503
