"""Request records and host-side synthetic traces (pkg/src/greengate/workload.py).

Traces are generated on the host with numpy's PCG64 streams in exactly the
reference's draw order (workload.py:87-171) — never on the device — so a
seed yields the same requests as the reference.  `generate_trace` returns
columnar numpy arrays (arrival times, [N, K] fp64 scores, labels) ready to be
pinned and copied into HBM; `generate_requests` returns the reference's
`RequestFeatures` list.  Checked against reference fixtures in
tests/test_workload.py.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from enum import Enum

import numpy as np

from .errors import ConfigError


class ArrivalMode(Enum):
    POISSON = "POISSON"
    ONOFF = "ONOFF"
    CLOSED = "CLOSED"


@dataclass(frozen=True)
class RequestFeatures:
    """One inference request as the controller sees it (workload.py:29-43)."""

    id: int
    arrival_t: float
    scores: tuple
    true_label: int | None = None

    def top_class(self) -> int:
        return max(range(len(self.scores)), key=self.scores.__getitem__)


@dataclass(frozen=True)
class WorkloadConfig:
    """workload.py:46-84 (same fields, defaults and validation)."""

    mode: ArrivalMode = ArrivalMode.POISSON
    rate_rps: float = 50.0
    on_rate_rps: float = 100.0
    off_rate_rps: float = 10.0
    phase_mean_s: float = 1.0
    num_requests: int = 100
    num_classes: int = 2
    confidence_low: float = 0.85
    confidence_high: float = 0.97
    fallback_degradation: float = 0.05
    seed: int | None = None

    def __post_init__(self) -> None:
        if self.num_classes < 2:
            raise ConfigError(f"num_classes must be >= 2, got {self.num_classes}")
        lo, hi = self.confidence_low, self.confidence_high
        if not (0.0 < lo <= hi <= 1.0):
            raise ConfigError(f"need 0 < confidence_low <= confidence_high <= 1, got {lo}, {hi}")
        if lo < 1.0 / self.num_classes:
            raise ConfigError(f"confidence_low {lo} below uniform score 1/{self.num_classes}")
        if not 0.0 <= self.fallback_degradation <= 1.0:
            raise ConfigError(
                f"fallback_degradation must be in [0, 1], got {self.fallback_degradation}")
        if self.mode is ArrivalMode.CLOSED and self.num_requests < 1:
            raise ConfigError(f"num_requests must be >= 1, got {self.num_requests}")
        if self.mode is ArrivalMode.POISSON and self.rate_rps <= 0.0:
            raise ConfigError(f"rate_rps must be > 0, got {self.rate_rps}")
        if self.mode is ArrivalMode.ONOFF:
            if self.on_rate_rps < 0.0 or self.off_rate_rps < 0.0:
                raise ConfigError("on/off rates must be >= 0")
            if self.phase_mean_s <= 0.0:
                raise ConfigError(f"phase_mean_s must be > 0, got {self.phase_mean_s}")


def _renewal_times(start: float, end: float, mean_gap: float, rng: np.random.Generator,
                   chunk: int = 4096) -> np.ndarray:
    """Times t_i = t_{i-1} + Exp(mean_gap) in [start, end), drawing exactly the
    variates the reference loop draws (workload.py:93-98, 133-139).

    Bulk `exponential(size=m)` yields the same variates as m scalar calls, and
    np.add.accumulate is a sequential left-to-right sum, so the times are
    bit-identical; the generator is rewound so it ends where the reference's
    does (one variate past the last accepted time).
    """
    out = []
    t = start
    while True:
        saved = rng.bit_generator.state
        xs = rng.exponential(mean_gap, size=chunk)
        acc = np.add.accumulate(np.concatenate(([t], xs)))[1:]
        over = np.nonzero(acc >= end)[0]
        if over.size == 0:
            out.append(acc)
            t = float(acc[-1])
            continue
        cut = int(over[0])
        rng.bit_generator.state = saved
        rng.exponential(mean_gap, size=cut + 1)
        out.append(acc[:cut])
        return np.concatenate(out) if out else np.empty(0)


def poisson_arrivals(rate_rps: float, horizon_s: float, rng: np.random.Generator) -> list[float]:
    if rate_rps <= 0.0:
        raise ConfigError(f"rate must be > 0, got {rate_rps}")
    return [float(x) for x in _renewal_times(0.0, horizon_s, 1.0 / rate_rps, rng)]


def onoff_phases(config: WorkloadConfig, horizon_s: float,
                 rng: np.random.Generator) -> list[tuple[float, float, float]]:
    phases = []
    t = 0.0
    on = True
    while t < horizon_s:
        length = float(rng.exponential(config.phase_mean_s))
        end = min(t + length, horizon_s)
        phases.append((t, end, config.on_rate_rps if on else config.off_rate_rps))
        t += length
        on = not on
    return phases


def onoff_arrivals(config: WorkloadConfig, horizon_s: float, rng: np.random.Generator) -> list[float]:
    times: list[np.ndarray] = []
    for start, end, rate in onoff_phases(config, horizon_s, rng):
        if rate <= 0.0:
            continue
        times.append(_renewal_times(start, end, 1.0 / rate, rng))
    return [float(x) for x in np.concatenate(times)] if times else []


@dataclass
class Trace:
    """Columnar trace: arrival_t [N] (NaN in CLOSED mode), scores [N, K] fp64,
    top_class [N], true_label [N]."""

    arrival_t: np.ndarray
    scores: np.ndarray
    top_class: np.ndarray
    true_label: np.ndarray

    def __len__(self) -> int:
        return int(self.scores.shape[0])

    def request(self, i: int) -> RequestFeatures:
        return RequestFeatures(int(i), float(self.arrival_t[i]),
                               tuple(float(x) for x in self.scores[i]), int(self.true_label[i]))


def _synth(n: int, config: WorkloadConfig, rng: np.random.Generator):
    """synth_request draws for n requests in order (workload.py:138-155)."""
    k = config.num_classes
    lo, hi = config.confidence_low, config.confidence_high
    c = np.empty(n)
    top = np.empty(n, np.int64)
    label = np.empty(n, np.int64)
    uniform, integers, random = rng.uniform, rng.integers, rng.random
    for i in range(n):
        ci = float(uniform(lo, hi))
        ti = int(integers(k))
        if float(random()) < ci:
            li = ti
        else:
            other = int(integers(k - 1))
            li = other if other < ti else other + 1
        c[i] = ci
        top[i] = ti
        label[i] = li
    rest = (1.0 - c) / (k - 1)
    scores = np.repeat(rest[:, None], k, axis=1)
    scores[np.arange(n), top] = c
    return scores, top, label


def generate_trace(config: WorkloadConfig, horizon_s: float, rng: np.random.Generator) -> Trace:
    """generate_requests (workload.py:158-171) as columnar arrays."""
    if config.mode is ArrivalMode.CLOSED:
        n = config.num_requests
        times = np.full(n, math.nan)
    elif config.mode is ArrivalMode.POISSON:
        if config.rate_rps <= 0.0:
            raise ConfigError(f"rate must be > 0, got {config.rate_rps}")
        times = _renewal_times(0.0, horizon_s, 1.0 / config.rate_rps, rng)
        n = times.shape[0]
    else:
        times = np.asarray(onoff_arrivals(config, horizon_s, rng), dtype=np.float64)
        n = times.shape[0]
    scores, top, label = _synth(n, config, rng)
    return Trace(times, scores, top, label)


def generate_requests(config: WorkloadConfig, horizon_s: float,
                      rng: np.random.Generator) -> list[RequestFeatures]:
    tr = generate_trace(config, horizon_s, rng)
    return [tr.request(i) for i in range(len(tr))]


def synth_request(req_id: int, arrival_t: float, config: WorkloadConfig,
                  rng: np.random.Generator) -> RequestFeatures:
    scores, _top, label = _synth(1, config, rng)
    return RequestFeatures(req_id, arrival_t, tuple(float(x) for x in scores[0]), int(label[0]))
