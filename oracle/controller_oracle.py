"""CPU restatement of the reference admission controller — TEST INFRASTRUCTURE.

This module is the parity oracle for the B200 hot path.  It is
imported only by `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` legs, and only as the checker: the
product path (`paper_2601_04250_b200`) never imports it and fails loudly when
its CUDA library is missing.

It restates, in plain CPython fp64, the arithmetic of
`/root/reference/pkg/src/greengate/controller.py`, `energy.py` and
`telemetry.percentile_nearest_rank` in the reference's operation order.  The
reference is not needed at run time; it is pinned against the reference's own
known-answer tests and against outputs of the reference captured in
`tests/golden/` by `tests/golden/make_golden.py` (run in the build container,
where `/root/reference` exists).

Summation follows CPython 3.12's `sum()` over floats (Neumaier compensation),
restated explicitly in `neumaier_sum` so the oracle does not depend on the
interpreter version; `tests/test_oracle.py` checks it against `sum()`.
"""

from __future__ import annotations

import math
from collections import deque
from dataclasses import dataclass, field
from typing import Iterable, Sequence

# Reference enum values (controller.py:38-64) as plain ints shared with the C ABI.
GEQ, LT = 0, 1
ENTROPY, ONE_MINUS_CONFIDENCE = 0, 1
ALL_DIRECT, ALL_BATCHED, THRESHOLD_ON_QUEUE = 0, 1, 2
SKIP, DIRECT, BATCHED, INVALID = 0, 1, 2, 255


class OracleInvalidDistribution(ValueError):
    """controller.py:129-134 raises InvalidDistribution."""


class OracleNegativeMeasurement(ValueError):
    """controller.py:347-353 / energy.py:33,81 raise NegativeMeasurement."""


def neumaier_sum(xs: Iterable[float]) -> float:
    """CPython >= 3.12 `sum()` of floats (Objects/bltinmodule.c builtin_sum_impl).

    Used by `_validate_distribution` (controller.py:132) and `entropy_utility`
    (controller.py:141).
    """
    s = 0.0
    c = 0.0
    for x in xs:
        t = s + x
        if abs(s) >= abs(x):
            c += (s - t) + x
        else:
            c += (x - t) + s
        s = t
    if c != 0.0 and math.isfinite(c):
        s += c
    return s


def validate_distribution(scores: Sequence[float]) -> list[float]:
    """controller.py:126-135."""
    xs = [float(s) for s in scores]
    if len(xs) < 2:
        raise OracleInvalidDistribution(f"need at least 2 class scores, got {len(xs)}")
    for x in xs:
        if not math.isfinite(x) or x < 0.0:
            raise OracleInvalidDistribution(f"scores must be finite and >= 0: {xs}")
    total = neumaier_sum(xs)
    if abs(total - 1.0) > 1e-9:
        raise OracleInvalidDistribution(f"scores must sum to 1 (got {total!r})")
    return xs


def _clamp01(v: float) -> float:
    """`min(1.0, max(0.0, v))` with Python's first-argument-wins tie rule."""
    v = v if v > 0.0 else 0.0
    return v if v < 1.0 else 1.0


def entropy_utility(scores: Sequence[float]) -> float:
    """controller.py:138-142: normalized Shannon entropy."""
    xs = validate_distribution(scores)
    h = -neumaier_sum(p * math.log(p) for p in xs if p > 0.0)
    return _clamp01(h / math.log(len(xs)))


def one_minus_confidence_utility(scores: Sequence[float]) -> float:
    """controller.py:145-148."""
    xs = validate_distribution(scores)
    return 1.0 - max(xs)


def utility(proxy: int, scores: Sequence[float]) -> float:
    """_UTILITY_FN dispatch (controller.py:151-154)."""
    if proxy == ENTROPY:
        return entropy_utility(scores)
    return one_minus_confidence_utility(scores)


def threshold_at(tau0: float, tau_inf: float, k: float, t_origin: float, t: float) -> float:
    """controller.py:114-123."""
    elapsed = t - t_origin
    elapsed = elapsed if elapsed > 0.0 else 0.0  # max(0.0, x)
    return tau_inf + (tau0 - tau_inf) * math.exp(-k * elapsed)


def cost(alpha: float, beta: float, gamma: float, u: float, e: float, c: float) -> float:
    """controller.py:214-216, left to right."""
    return alpha * u + beta * e + gamma * c


def admits(direction: int, composite: float, threshold: float) -> bool:
    """Direction.admits (controller.py:44-47)."""
    if direction == GEQ:
        return composite >= threshold
    return composite < threshold


def ewma_update(prev: float | None, sample: float, lam: float) -> float:
    """energy.py:24-36."""
    if prev is None:
        return sample
    return lam * prev + (1.0 - lam) * sample


def percentile_nearest_rank(values: Sequence[float], p: float) -> float:
    """telemetry.py:35-46."""
    ordered = sorted(values)
    rank = math.ceil(p / 100.0 * len(ordered))
    return ordered[rank - 1]


@dataclass
class Channel:
    """NormalizerChannel (controller.py:157-183); None == unseen."""

    lo: float | None = None
    hi: float | None = None

    def observe(self, raw: float) -> None:
        if self.lo is None or raw < self.lo:
            self.lo = raw
        if self.hi is None or raw > self.hi:
            self.hi = raw

    def normalize(self, raw: float) -> float:
        self.observe(raw)
        lo, hi = self.lo, self.hi
        if hi <= lo:
            return 0.0
        return _clamp01((raw - lo) / (hi - lo))


@dataclass
class OracleParams:
    alpha: float = 1.0
    beta: float = 0.0
    gamma: float = 0.0
    tau0: float = 1.0
    tau_inf: float = 0.2
    k: float = 0.5
    ewma_lambda: float = 0.9
    direction: int = GEQ
    utility_proxy: int = ENTROPY
    routing: int = ALL_DIRECT
    queue_threshold: int = 4
    p95_window: int = 100


@dataclass
class OracleDecision:
    code: int            # SKIP / DIRECT / BATCHED
    utility: float
    energy: float
    congestion: float
    composite: float
    threshold: float

    @property
    def admit(self) -> bool:
        return self.code in (DIRECT, BATCHED)


@dataclass
class OracleController:
    """AdmissionController state machine (controller.py:256-362)."""

    params: OracleParams = field(default_factory=OracleParams)
    t_origin: float = 0.0
    energy: Channel = field(default_factory=Channel)
    queue: Channel = field(default_factory=Channel)
    p95: Channel = field(default_factory=Channel)
    ewma: float = 0.0
    samples_seen: int = 0
    total_joules: float = 0.0
    admitted_total: int = 0
    skipped_total: int = 0
    queue_depth: int = 0          # default congestion source reports 0
    latencies: deque = None       # type: ignore[assignment]

    def __post_init__(self) -> None:
        if self.latencies is None:
            self.latencies = deque(maxlen=self.params.p95_window)

    def p95_ms(self) -> float:
        """controller.py:289-293."""
        if not self.latencies:
            return 0.0
        return percentile_nearest_rank(list(self.latencies), 95.0)

    def default_snapshot(self) -> tuple[int, float, float]:
        """controller.py:295-300 with the gateway's reported depth."""
        return (self.queue_depth, self.p95_ms(), 0.0)

    def _route(self, queue_depth: int) -> int:
        """controller.py:302-307."""
        r = self.params.routing
        if r == ALL_BATCHED:
            return BATCHED
        if r == THRESHOLD_ON_QUEUE:
            return BATCHED if queue_depth > self.params.queue_threshold else DIRECT
        return DIRECT

    def decide(self, scores: Sequence[float], now: float,
               snapshot: tuple[int, float, float] | None = None) -> OracleDecision:
        """controller.py:309-343.  Raises OracleInvalidDistribution with no state change."""
        p = self.params
        u = utility(p.utility_proxy, scores)
        if self.samples_seen > 0:
            e = self.energy.normalize(self.ewma)
        else:
            e = 0.0
        qd, p95v, fill = snapshot if snapshot is not None else self.default_snapshot()
        c = (self.queue.normalize(float(qd)) + self.p95.normalize(p95v) + fill) / 3.0
        j = cost(p.alpha, p.beta, p.gamma, u, e, c)
        tau = threshold_at(p.tau0, p.tau_inf, p.k, self.t_origin, now)
        if admits(p.direction, j, tau):
            code = self._route(qd)
            self.admitted_total += 1
        else:
            code = SKIP
            self.skipped_total += 1
        return OracleDecision(code, u, e, c, j, tau)

    def decide_batch(self, rows: Sequence[Sequence[float]], nows: Sequence[float],
                     snapshot: tuple[int, float, float] | None = None):
        """Sequential decide() over a micro-batch with one frozen snapshot.

        Invalid rows are reported as INVALID and skipped, which is what a caller
        looping over decide() and catching InvalidDistribution observes.
        """
        snap = snapshot if snapshot is not None else self.default_snapshot()
        out = []
        for row, now in zip(rows, nows):
            try:
                out.append(self.decide(row, now, snap))
            except OracleInvalidDistribution:
                out.append(None)
        return out

    def record_outcome(self, latency_ms: float, joules: float, queue_depth: int) -> None:
        """controller.py:345-358 (+ EnergyLedger.observe_request energy.py:75-87)."""
        if latency_ms < 0.0 or joules < 0.0 or queue_depth < 0:
            raise OracleNegativeMeasurement(
                f"latency={latency_ms!r} joules={joules!r} depth={queue_depth!r}")
        prev = self.ewma if self.samples_seen > 0 else None
        self.ewma = ewma_update(prev, joules, self.params.ewma_lambda)
        self.samples_seen += 1
        self.total_joules += joules
        self.latencies.append(latency_ms)
        self.energy.observe(self.ewma)
        self.queue.observe(float(queue_depth))
        self.p95.observe(self.p95_ms())

    def reset_clock(self, t_origin: float) -> None:
        """controller.py:360-362."""
        self.t_origin = t_origin

    def state_tuple(self) -> dict:
        """Comparable view of the loop state (matches gg_state fields)."""
        def ch(c: Channel):
            return (c.lo, c.hi) if c.lo is not None else None
        return {
            "energy": ch(self.energy), "queue_depth": ch(self.queue), "p95_ms": ch(self.p95),
            "ewma": self.ewma, "samples_seen": self.samples_seen,
            "total_joules": self.total_joules,
            "admitted_total": self.admitted_total, "skipped_total": self.skipped_total,
            "p95_current": self.p95_ms(), "t_origin": self.t_origin,
        }


def softmax_fp64(logits: Sequence[float]) -> list[float]:
    """Oracle for the K3 epilogue: fp32 logits widened to fp64, max-shifted
    softmax in fp64 (no reference symbol; consumers are RequestFeatures.scores,
    workload.py:29-43).  Sum order: left to right, plain (what the kernel does)."""
    xs = [float(x) for x in logits]
    m = max(xs)
    ex = [math.exp(x - m) for x in xs]
    s = 0.0
    for v in ex:
        s += v
    return [v / s for v in ex]


def top_class(scores: Sequence[float]) -> int:
    """RequestFeatures.top_class (workload.py:42-43): first index of the max."""
    return max(range(len(scores)), key=scores.__getitem__)
