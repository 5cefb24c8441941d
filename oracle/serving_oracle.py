"""Host replay of the closed serving loop with the C restatement — TEST INFRASTRUCTURE.

Mirrors paper_2601_04250_b200.serving.GatedServer step by step with the C
oracle standing in for K1/K2 (the forward does not affect the controller):

  snapshot = (fifo depth + other ranks' depth, p95, min(1, depth / B))   servesim.py:211-220
  decide window rows with that frozen snapshot                           controller.py:309-343
  append admitted rows to the FIFO, pop up to B                          servesim.py:286-306
  outcomes: latency = base + per_item * n, joules = (base_j + per_item_j * n) / n,
            queue depth = depth after the pop (+ other ranks' depth)     servesim.py:303-304
  record_outcome for every served request of every rank in rank order    controller.py:345-358

Data-parallel semantics (G ranks, one replicated controller): within a step
every rank decides its window against the same replicated state S with its
own snapshot; the step's state is S plus every rank's admission effects
(normalizer observes of its snapshot, counters — all commutative) followed by
all ranks' outcomes in rank order.  With G = 1 this is exactly sequential
decide()/record_outcome().
"""

from __future__ import annotations

import ctypes as C
from collections import deque

import numpy as np

from paper_2601_04250_b200 import _abi

from . import c_oracle


def _copy_state(s: _abi.gg_state) -> _abi.gg_state:
    return _abi.gg_state.from_buffer_copy(bytes(s))


def _merge_channel(dst: _abi.gg_channel, src: _abi.gg_channel) -> None:
    if not src.seen:
        return
    if not dst.seen or src.lo < dst.lo:
        dst.lo = src.lo
    if not dst.seen or src.hi > dst.hi:
        dst.hi = src.hi
    dst.seen = 1


def _observe(ch: _abi.gg_channel, raw: float) -> None:
    """NormalizerChannel.observe (controller.py:164-170)."""
    if not ch.seen or raw < ch.lo:
        ch.lo = raw
    if not ch.seen or raw > ch.hi:
        ch.hi = raw
    ch.seen = 1


def _open_admit(params, state, qd: int, p95: float, n: int) -> int:
    """Open-loop arm (servesim.py:231-240): static route; the state gets the
    counters and snapshot observes of an always-admitting decide()."""
    if n > 0:
        if state.samples_seen > 0:
            _observe(state.n_energy, state.ewma_joules_per_request)
        _observe(state.n_queue_depth, float(qd))
        _observe(state.n_p95_ms, p95)
        state.admitted_total += n
    if params.routing == _abi.GG_ROUTE_ALL_BATCHED:
        return _abi.GG_DECISION_BATCHED
    if params.routing == _abi.GG_ROUTE_THRESHOLD_ON_QUEUE and qd > params.queue_threshold:
        return _abi.GG_DECISION_BATCHED
    return _abi.GG_DECISION_DIRECT


def replay(params, shards, window: int, B: int, model: dict, steps: int, *,
           open_loop: bool = False, window_s: float | None = None, latency: str = "model",
           labels=None, coins=None, degradation: float = 0.05, records: dict | None = None):
    """shards: list of (scores [T_g, K], now [T_g]) per rank.  Returns per-rank
    decisions (trace indexed), per-rank served order, and the final state.

    open_loop: controller disabled (servesim.py:231-240).  window_s: Path-B
    flush policy in trace time (servesim.py:148-162).  latency "trace": the
    reference's finish - enqueue.  labels/coins (per rank lists): fallback
    accounting (servesim.py:246-256); with `records` (a dict) the per-rank
    answer / correct / latency columns are returned in it."""
    G = len(shards)
    state = c_oracle.COracle(params).state
    fifos = [deque() for _ in range(G)]
    cursors = [0] * G
    clocks = [0.0] * G
    coin_cur = [0] * G
    extra = [0] * G
    decisions = [np.full(s[0].shape[0], 254, np.uint8) for s in shards]
    served = [[] for _ in range(G)]
    cols = [dict(answer=np.full(s[0].shape[0], -1, np.int32),
                 correct=np.zeros(s[0].shape[0], np.uint8),
                 latency=np.zeros(s[0].shape[0], np.float64)) for s in shards]
    trace_clock = window_s is not None or latency == "trace"
    for _ in range(steps):
        base = _copy_state(state)
        after = []
        slots = []
        for g, (scores, now) in enumerate(shards):
            orc = c_oracle.COracle(params)
            orc.state = _copy_state(base)
            depth = len(fifos[g])
            snap = (depth + extra[g], base.p95_current, min(1.0, depth / B))
            T = scores.shape[0]
            c0 = cursors[g]
            c1 = min(T, c0 + window)
            if c1 > c0:
                if open_loop:
                    code = _open_admit(params, orc.state, snap[0], snap[1], c1 - c0)
                    dec = np.full(c1 - c0, code, np.uint8)
                    idx = np.arange(c1 - c0)
                else:
                    dec, _bd, idx, _info = orc.admit(scores[c0:c1], now[c0:c1], snap,
                                                     want_breakdown=False)
                decisions[g][c0:c1] = dec
                fifos[g].extend(int(c0 + i) for i in idx)
                if labels is not None:
                    for r in range(c0, c1):
                        d = int(decisions[g][r])
                        if d == _abi.GG_DECISION_INVALID:
                            continue
                        top = int(np.argmax(scores[r]))          # first max (workload.py:42-43)
                        cols[g]["answer"][r] = top
                        hit = top == int(labels[g][r])
                        if d == _abi.GG_DECISION_SKIP:
                            ok = False
                            if hit:                               # `and` short-circuits the coin
                                ok = float(coins[g][coin_cur[g]]) >= degradation
                                coin_cur[g] += 1
                        else:
                            ok = hit
                        cols[g]["correct"][r] = int(ok)
            cursors[g] = c1
            after.append(orc.state)
            depth = len(fifos[g])
            n = min(B, depth)
            if trace_clock:
                cur = min(cursors[g], T)
                clock = float(now[cur - 1]) if cur > 0 else 0.0
                if window_s is not None and window_s > 0.0 and 0 < depth < B:
                    oldest = float(now[fifos[g][0]])
                    if cursors[g] >= T:
                        clock = max(clock, oldest + window_s)
                    elif not (clock - oldest >= window_s - 1e-12):
                        n = 0
                clocks[g] = max(clocks[g], clock)
            batch = [fifos[g].popleft() for _ in range(n)]
            served[g].extend(batch)
            dn = float(n if n > 0 else 1)
            lat_m = model["batch_base_ms"] + model["per_item_ms"] * dn
            jo = (model["batch_base_energy_j"] + model["per_item_energy_j"] * dn) / dn
            if latency == "trace":
                finish = clocks[g] + lat_m / 1000.0
                lats = np.array([(finish - float(now[r])) * 1000.0 for r in batch], np.float64)
            else:
                lats = np.full(n, lat_m)
            cols[g]["latency"][batch] = lats
            slots.append((n, lats, jo, len(fifos[g]) + extra[g], len(fifos[g])))
        # admission effects of every rank (commutative)
        for s in after:
            for name in ("n_energy", "n_queue_depth", "n_p95_ms"):
                _merge_channel(getattr(state, name), getattr(s, name))
            state.admitted_total += s.admitted_total - base.admitted_total
            state.skipped_total += s.skipped_total - base.skipped_total
        # outcomes in rank order
        orc = c_oracle.COracle(params)
        orc.state = state
        for n, lats, jo, qd, _d in slots:
            if n:
                orc.outcome(lats, np.full(n, jo), np.full(n, qd, np.int32),
                            set_queue_depth=True)
        state = orc.state
        for g in range(G):
            extra[g] = sum(s[4] for h, s in enumerate(slots) if h != g)
    if records is not None:
        records["columns"] = cols
        records["coin_cursor"] = coin_cur
        records["clock"] = clocks
    return decisions, served, state


def state_bytes_equal(a: _abi.gg_state, b: _abi.gg_state) -> bool:
    return bytes(a) == bytes(b)


__all__ = ["replay", "state_bytes_equal", "C"]
