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


def replay(params, shards, window: int, B: int, model: dict, steps: int):
    """shards: list of (scores [T_g, K], now [T_g]) per rank.  Returns per-rank
    decisions (trace indexed), per-rank served order, and the final state."""
    G = len(shards)
    state = c_oracle.COracle(params).state
    fifos = [deque() for _ in range(G)]
    cursors = [0] * G
    extra = [0] * G
    decisions = [np.full(s[0].shape[0], 254, np.uint8) for s in shards]
    served = [[] for _ in range(G)]
    for _ in range(steps):
        base = _copy_state(state)
        after = []
        slots = []
        for g, (scores, now) in enumerate(shards):
            orc = c_oracle.COracle(params)
            orc.state = _copy_state(base)
            depth = len(fifos[g])
            snap = (depth + extra[g], base.p95_current, min(1.0, depth / B))
            c0 = cursors[g]
            c1 = min(scores.shape[0], c0 + window)
            if c1 > c0:
                dec, _bd, idx, _info = orc.admit(scores[c0:c1], now[c0:c1], snap,
                                                 want_breakdown=False)
                decisions[g][c0:c1] = dec
                fifos[g].extend(int(c0 + i) for i in idx)
            cursors[g] = c1
            after.append(orc.state)
            n = min(B, len(fifos[g]))
            served[g].extend(fifos[g].popleft() for _ in range(n))
            dn = float(n if n > 0 else 1)
            lat = model["batch_base_ms"] + model["per_item_ms"] * dn
            jo = (model["batch_base_energy_j"] + model["per_item_energy_j"] * dn) / dn
            slots.append((n, lat, jo, len(fifos[g]) + extra[g], len(fifos[g])))
        # admission effects of every rank (commutative)
        for s in after:
            for name in ("n_energy", "n_queue_depth", "n_p95_ms"):
                _merge_channel(getattr(state, name), getattr(s, name))
            state.admitted_total += s.admitted_total - base.admitted_total
            state.skipped_total += s.skipped_total - base.skipped_total
        # outcomes in rank order
        orc = c_oracle.COracle(params)
        orc.state = state
        for n, lat, jo, qd, _d in slots:
            if n:
                orc.outcome(np.full(n, lat), np.full(n, jo), np.full(n, qd, np.int32),
                            set_queue_depth=True)
        state = orc.state
        for g in range(G):
            extra[g] = sum(s[4] for h, s in enumerate(slots) if h != g)
    return decisions, served, state


def state_bytes_equal(a: _abi.gg_state, b: _abi.gg_state) -> bool:
    return bytes(a) == bytes(b)


__all__ = ["replay", "state_bytes_equal", "C"]
