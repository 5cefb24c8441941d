"""Closed serving loop on the GPU vs the host replay (oracle/serving_oracle.py).

Checks, for ResNet-18 (K=1000 gating scores) and DistilBERT (K=2) loops:
  - every trace row's decision code equals the oracle's (bit-exact outside the
    |J - tau| < 1e-12 band; the fixtures have no such rows),
  - the served order (FIFO) and the set of served requests equal the oracle's,
  - the controller state after the loop equals the oracle's field by field,
  - graph replay == eager steps.
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import serving_oracle
from tests import _golden as G

pytestmark = pytest.mark.gpu

MODEL = dict(batch_base_ms=4.0, per_item_ms=0.05, batch_base_energy_j=6.0, per_item_energy_j=1.5)


def make_trace(n, k, seed):
    import paper_2601_04250_b200 as gg
    wl = gg.WorkloadConfig(mode=gg.ArrivalMode.POISSON, rate_rps=5000.0, num_classes=k,
                           confidence_low=max(0.3, 1.0 / k), confidence_high=0.95)
    tr = gg.generate_trace(wl, 10.0, np.random.default_rng(seed))
    return tr.scores[:n].copy(), tr.arrival_t[:n].copy()


def build(kind, B, window, scores, now, cfg_kw, graph):
    import torch
    import paper_2601_04250_b200 as gg
    from paper_2601_04250_b200 import serving
    cfg = gg.ControllerConfig(**cfg_kw)
    ctl = cfg.build(gg.EnergyLedger())
    if kind == "resnet18":
        from paper_2601_04250_b200.resnet18 import ResNet18B200, random_model
        net = ResNet18B200(random_model(0), max_batch=B)
        payloads = serving.synthetic_images(32)
    else:
        from paper_2601_04250_b200.distilbert import DistilBertB200, random_model
        net = DistilBertB200(random_model(0), max_batch=B)
        payloads = serving.synthetic_tokens(32)
    srv = serving.GatedServer(ctl, net, torch.from_numpy(scores).cuda(),
                              torch.from_numpy(now).cuda(), payloads, window=window,
                              outcome=serving.OutcomeModel(**MODEL), fifo_capacity=4096)
    srv.run(1)
    if graph:
        srv.capture()
    return srv, cfg


@pytest.mark.parametrize("kind,k,B,window,graph", [
    ("resnet18", 1000, 16, 24, True), ("resnet18", 1000, 8, 8, False), ("distilbert", 2, 16, 40, True)])
def test_serving_loop_vs_oracle(kind, k, B, window, graph):
    import torch
    n = 600 if kind == "distilbert" else 300
    scores, now = make_trace(n, k, seed=k)
    cfg_kw = dict(alpha=1.0, beta=-0.2, gamma=-0.4, tau0=0.8, tau_inf=0.35, k=1.5,
                  routing=__import__("paper_2601_04250_b200").RoutePolicy.ALL_BATCHED)
    srv, cfg = build(kind, B, window, scores, now, cfg_kw, graph)
    steps = 1
    while not srv.done():
        srv.run(1)
        steps += 1
        assert steps < 10_000
    torch.cuda.synchronize()
    p = G.abi_params(dict(alpha=1.0, beta=-0.2, gamma=-0.4, tau0=0.8, tau_inf=0.35, k=1.5,
                          ewma_lambda=0.9, direction=0, utility_proxy=0, routing=1,
                          queue_threshold=4, p95_window=100))
    dec_o, served_o, st_o = serving_oracle.replay(p, [(scores, now)], window, B, MODEL, steps)
    dec = srv.decision.cpu().numpy()
    assert np.array_equal(dec, dec_o[0])
    pred = srv.predicted.cpu().numpy()
    assert set(np.nonzero(pred >= 0)[0]) == set(served_o[0])
    r = srv.results()
    assert r["overflow"] == 0 and r["served"] == len(served_o[0])
    got = G.state_dict_of_abi(srv.ctl.state_struct())
    want = G.state_dict_of_abi(st_o)
    assert got == want
    conf = srv.confidence.cpu().numpy()[pred >= 0]
    assert ((conf > 0) & (conf <= 1)).all()


def _labels(n, k, seed):
    rng = np.random.default_rng(seed)
    return rng.integers(0, k, size=n).astype(np.int32)


@pytest.mark.parametrize("kind,k,B,window,open_loop,win_ms,latency,routing", [
    ("distilbert", 2, 16, 40, False, 6.0, "trace", 1),     # Path-B flush + queueing latency
    ("distilbert", 2, 16, 40, True, 6.0, "trace", 2),      # open-loop arm, THRESHOLD_ON_QUEUE
    ("distilbert", 2, 16, 24, True, None, "model", 0),     # open-loop, size trigger only
    ("resnet18", 1000, 8, 12, False, 4.0, "trace", 2),
    ("resnet18", 1000, 8, 12, True, 4.0, "model", 1),
])
def test_serving_policies_vs_oracle(kind, k, B, window, open_loop, win_ms, latency, routing):
    """Open-loop arm (servesim.py:231-240), Path-B flush policy (148-162), trace-time
    latency (finish - enqueue) and the fallback answers / accuracy accounting
    (246-256) on the device loop == the host replay, row for row, and the final
    controller state byte-equal."""
    import torch
    import paper_2601_04250_b200 as gg
    from paper_2601_04250_b200 import serving
    n = 500 if kind == "distilbert" else 200
    scores, now = make_trace(n, k, seed=k + 3)
    labels = _labels(n, k, seed=9)
    coins = serving.fallback_coins(123, n)
    deg = 0.2
    cfg_kw = dict(alpha=1.0, beta=-0.2, gamma=-0.4, tau0=0.8, tau_inf=0.35, k=1.5,
                  routing=[gg.RoutePolicy.ALL_DIRECT, gg.RoutePolicy.ALL_BATCHED,
                           gg.RoutePolicy.THRESHOLD_ON_QUEUE][routing], queue_threshold=6)
    # the open-loop arm comes from the config's `enabled`, as in the reference simulator
    ctl = gg.ControllerConfig(enabled=not open_loop, **cfg_kw).build(gg.EnergyLedger())
    if kind == "resnet18":
        from paper_2601_04250_b200.resnet18 import ResNet18B200, random_model
        net = ResNet18B200(random_model(0), max_batch=B)
        payloads = serving.synthetic_images(32)
    else:
        from paper_2601_04250_b200.distilbert import DistilBertB200, random_model
        net = DistilBertB200(random_model(0), max_batch=B)
        payloads = serving.synthetic_tokens(32)
    srv = serving.GatedServer(
        ctl, net, torch.from_numpy(scores).cuda(), torch.from_numpy(now).cuda(), payloads,
        window=window, outcome=serving.OutcomeModel(**MODEL, latency=latency), fifo_capacity=4096,
        batching_window_ms=win_ms, labels=torch.from_numpy(labels).cuda(),
        coins=torch.from_numpy(coins).cuda(), fallback_degradation=deg)
    assert srv.open_loop == open_loop
    srv.run(1)
    srv.capture()
    steps = 1
    while not srv.done():
        srv.run(1)
        steps += 1
        assert steps < 10_000
    torch.cuda.synchronize()
    p = G.abi_params(dict(alpha=1.0, beta=-0.2, gamma=-0.4, tau0=0.8, tau_inf=0.35, k=1.5,
                          ewma_lambda=0.9, direction=0, utility_proxy=0, routing=routing,
                          queue_threshold=6, p95_window=100))
    rec = {}
    dec_o, served_o, st_o = serving_oracle.replay(
        p, [(scores, now)], window, B, MODEL, steps, open_loop=open_loop,
        window_s=None if win_ms is None else win_ms / 1000.0, latency=latency, labels=[labels],
        coins=[coins], degradation=deg, records=rec)
    dec = srv.decision.cpu().numpy()
    assert np.array_equal(dec, dec_o[0])
    if open_loop:
        assert (dec != 0).all()                       # admit everything
    cols = rec["columns"][0]
    assert np.array_equal(srv.answer.cpu().numpy(), cols["answer"])
    assert np.array_equal(srv.correct.cpu().numpy(), cols["correct"])
    assert int(srv.coin_cursor.item()) == rec["coin_cursor"][0]
    assert np.array_equal(srv.latency.cpu().numpy(), cols["latency"])   # bit-exact fp64
    pred = srv.predicted.cpu().numpy()
    assert set(np.nonzero(pred >= 0)[0]) == set(served_o[0])
    r = srv.results()
    assert r["overflow"] == 0 and r["served"] == len(served_o[0]) and r["clock"] == rec["clock"][0]
    st = srv.ctl.state_struct()
    assert G.state_dict_of_abi(st) == G.state_dict_of_abi(st_o)
    assert (st.outcomes_total, st.win_count, st.queue_depth) == \
        (st_o.outcomes_total, st_o.win_count, st_o.queue_depth)
    if open_loop:
        assert r["served"] == n
    s = srv.summary()
    assert s["admitted_count"] + s["skipped_count"] == n and 0.0 <= s["accuracy"] <= 1.0


@pytest.mark.parametrize("graph", [True, False])
def test_published_step_records(graph):
    """GatedServer(publish=True): each step's last kernel writes the served batch's
    predictions / confidences and the window's decisions into pinned host memory
    (gg_publish_step); the record of step i equals the device arrays after step i."""
    import torch
    import paper_2601_04250_b200 as gg
    from paper_2601_04250_b200 import serving
    from paper_2601_04250_b200.distilbert import DistilBertB200, random_model
    scores, now = make_trace(400, 2, seed=21)
    ctl = gg.ControllerConfig(alpha=1.0, beta=-0.2, gamma=-0.3, tau0=0.8, tau_inf=0.35,
                              k=1.5).build(gg.EnergyLedger())
    net = DistilBertB200(random_model(0), max_batch=16)
    srv = serving.GatedServer(ctl, net, torch.from_numpy(scores).cuda(),
                              torch.from_numpy(now).cuda(), serving.synthetic_tokens(32),
                              window=24, outcome=serving.OutcomeModel(**MODEL), publish=True)
    srv.run(1)
    if graph:
        srv.capture()
    c0 = 24
    for _ in range(12):
        srv.run(1)
        torch.cuda.synchronize()
        rec = srv.record(srv.steps_run - 1)
        n = int(srv.count.item())
        assert rec["count"] == n
        assert np.array_equal(rec["pred"], srv.batch_pred[:n].cpu().numpy())
        assert np.array_equal(rec["conf"], srv.batch_conf[:n].cpu().numpy())
        assert rec["window_start"] == c0
        assert np.array_equal(rec["decision"], srv.decision[c0:c0 + len(rec["decision"])].cpu().numpy())
        c0 += len(rec["decision"])
    with pytest.raises(RuntimeError):
        srv.record(srv.steps_run - 3)   # the slot has been reused


@pytest.mark.parametrize("k", [2, 1000])
def test_fallback_answers_large_window(k):
    """gg_fallback_answers over an explicit row range longer than one cluster
    super-chunk (4096 rows) and not starting at 0: answers = first-max top class
    (rows with tied maxima included), correct flags and the coin cursor == the
    reference accounting (servesim.py:246-256) replayed in numpy; invalid rows
    are left untouched."""
    import ctypes as C
    import torch
    from paper_2601_04250_b200 import _abi, _native
    lib = _native.load()
    rng = np.random.default_rng(k)
    T, row0, n = 9000, 37, 8500
    scores = rng.random((T, k))
    scores /= scores.sum(axis=1, keepdims=True)
    tie = rng.random(T) < 0.1                           # duplicated maxima: first max wins
    for r in np.nonzero(tie)[0]:
        m = int(np.argmax(scores[r]))
        scores[r, (m + 1 + rng.integers(0, k - 1)) % k] = scores[r, m]
    top = np.argmax(scores, axis=1)
    labels = np.where(rng.random(T) < 0.6, top, rng.integers(0, k, T)).astype(np.int32)
    codes = np.array([_abi.GG_DECISION_SKIP, _abi.GG_DECISION_DIRECT, _abi.GG_DECISION_BATCHED,
                      _abi.GG_DECISION_INVALID], np.uint8)
    dec = codes[rng.choice(4, T, p=[0.5, 0.2, 0.2, 0.1])]
    coins = rng.random(T)
    deg = 0.3
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    s_d, l_d, dec_d, c_d = d(scores), d(labels), d(dec), d(coins)
    ans = torch.full((T,), -7, dtype=torch.int32, device="cuda")
    cor = torch.full((T,), 9, dtype=torch.uint8, device="cuda")
    cur = torch.tensor([5], dtype=torch.int64, device="cuda")
    _native.check("gg_fallback_answers", lib.gg_fallback_answers(
        _native.ptr(s_d), k, k, _native.ptr(l_d), _native.ptr(dec_d), None, None, row0, n,
        _native.ptr(c_d), _native.ptr(cur), deg, _native.ptr(ans), _native.ptr(cor), None))
    torch.cuda.synchronize()
    want_a = np.full(T, -7, np.int32)
    want_c = np.full(T, 9, np.uint8)
    cc = 5
    for r in range(row0, row0 + n):
        if dec[r] == _abi.GG_DECISION_INVALID:
            continue
        want_a[r] = top[r]
        hit = top[r] == labels[r]
        if dec[r] == _abi.GG_DECISION_SKIP:
            ok = False
            if hit:
                ok = coins[cc] >= deg
                cc += 1
        else:
            ok = hit
        want_c[r] = ok
    assert np.array_equal(ans.cpu().numpy(), want_a)
    assert np.array_equal(cor.cpu().numpy(), want_c)
    assert int(cur.item()) == cc


@pytest.mark.parametrize("kind,k,B,window,win_ms,latency,open_loop", [
    ("distilbert", 2, 16, 24, None, "model", False),
    ("distilbert", 2, 16, 24, 4.0, "trace", False),
    ("distilbert", 2, 16, 40, 6.0, "trace", True),
    ("resnet18", 1000, 8, 12, 4.0, "trace", False),
])
def test_pipelined_steps_match_sequential(kind, k, B, window, win_ms, latency, open_loop):
    """GatedServer(pipeline=True) -- the control chain of step t+1 on the serving
    stream while step t's forward / K3 / publish run on a second stream, per-step
    buffers in two alternating sets, two parity graphs -- ends in exactly the
    sequential loop's state: decisions, fallback answers and accounting,
    predictions and confidences, latencies, FIFO counters, controller state and
    the last published record."""
    import torch
    import paper_2601_04250_b200 as gg
    from paper_2601_04250_b200 import serving
    n = 400 if kind == "distilbert" else 160
    scores, now = make_trace(n, k, seed=k + 11)
    labels = _labels(n, k, seed=4)
    coins = serving.fallback_coins(77, n)
    if kind == "resnet18":
        from paper_2601_04250_b200.resnet18 import ResNet18B200, random_model
        net_f = lambda: ResNet18B200(random_model(0), max_batch=B)   # noqa: E731
        payloads = serving.synthetic_images(32)
    else:
        from paper_2601_04250_b200.distilbert import DistilBertB200, random_model
        net_f = lambda: DistilBertB200(random_model(0), max_batch=B)   # noqa: E731
        payloads = serving.synthetic_tokens(32)
    out = {}
    for pipe in (False, True):
        ctl = gg.ControllerConfig(alpha=1.0, beta=-0.2, gamma=-0.4, tau0=0.8, tau_inf=0.35, k=1.5,
                                  routing=gg.RoutePolicy.THRESHOLD_ON_QUEUE,
                                  queue_threshold=6).build(gg.EnergyLedger())
        srv = serving.GatedServer(
            ctl, net_f(), torch.from_numpy(scores).cuda(), torch.from_numpy(now).cuda(), payloads,
            window=window, outcome=serving.OutcomeModel(**MODEL, latency=latency),
            fifo_capacity=4096, batching_window_ms=win_ms, labels=torch.from_numpy(labels).cuda(),
            coins=torch.from_numpy(coins).cuda(), fallback_degradation=0.2, publish=True,
            pipeline=pipe, open_loop=open_loop)
        srv.run(1)
        srv.capture()
        steps = 1
        while not srv.done():   # fifo_state() syncs the serving stream: exact step counts
            srv.run(1)
            steps += 1
            assert steps < 10_000
        torch.cuda.synchronize()
        out[pipe] = dict(
            arrays=[t.cpu().numpy() for t in (srv.decision, srv.answer, srv.correct, srv.predicted,
                                              srv.confidence, srv.latency, srv.coin_cursor)],
            results=srv.results(), state=G.state_dict_of_abi(srv.ctl.state_struct()),
            steps=srv.steps_run, control=srv.control_steps,
            last=srv.record(srv.steps_run - 1))
    a, b = out[False], out[True]
    for x, y in zip(a["arrays"], b["arrays"]):
        assert np.array_equal(x, y, equal_nan=x.dtype.kind == "f")
    assert a["results"] == b["results"] and a["state"] == b["state"]
    assert a["steps"] == b["steps"] == a["control"] == b["control"]
    for key in ("count", "window_start"):
        assert a["last"][key] == b["last"][key]
    for key in ("pred", "conf", "decision"):
        assert np.array_equal(a["last"][key], b["last"][key])


def test_measured_latency_feedback():
    """latency="measured": the served-outcome kernel stamps %globaltimer after the
    forward and K3, so each served request's latency (admission -> completion of its
    batch's epilogue) is the device's own and drives the controller on the device:
    the state's p95 equals the nearest-rank p95 (telemetry.py:35-46) of the last
    p95_window served latencies.  The pipelined loop refuses this mode (its control
    chain does not wait for the forward)."""
    import math
    import torch
    import paper_2601_04250_b200 as gg
    from paper_2601_04250_b200 import serving
    from paper_2601_04250_b200.distilbert import DistilBertB200, random_model
    n, B, window = 240, 16, 24
    scores, now = make_trace(n, 2, seed=21)
    ctl = gg.ControllerConfig(alpha=1.0, beta=-0.2, gamma=-0.4, tau0=0.8, tau_inf=0.35, k=1.5,
                              routing=gg.RoutePolicy.ALL_BATCHED).build(gg.EnergyLedger())
    net = DistilBertB200(random_model(0), max_batch=B)
    kw = dict(window=window, outcome=serving.OutcomeModel(**MODEL, latency="measured"),
              fifo_capacity=1024)
    with pytest.raises(ValueError):
        serving.GatedServer(ctl, net, torch.from_numpy(scores).cuda(), torch.from_numpy(now).cuda(),
                            serving.synthetic_tokens(32), pipeline=True, **kw)
    srv = serving.GatedServer(ctl, net, torch.from_numpy(scores).cuda(), torch.from_numpy(now).cuda(),
                              serving.synthetic_tokens(32), **kw)
    srv.run(1)
    srv.capture()
    while not srv.done():
        srv.run(1)
    torch.cuda.synchronize()
    pred = srv.predicted.cpu().numpy()
    lat = srv.latency.cpu().numpy()
    served = np.nonzero(pred >= 0)[0]                  # FIFO order == trace order
    assert len(served) > 10
    ls = lat[served]
    assert np.all(np.isfinite(ls)) and np.all(ls > 0.0)
    st = srv.ctl.state_struct()
    assert st.outcomes_total == len(served)
    last = np.sort(ls[-int(srv.ctl.params.p95_window):])
    k = max(1, math.ceil(0.95 * len(last)))
    assert st.p95_current == last[k - 1]
