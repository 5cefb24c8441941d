"""Device-backed admission controller — drop-in for pkg/src/greengate/controller.py.

Same public names, fields, defaults, enum values, method signatures and
exceptions as the reference module; the arithmetic runs in the sm_100a
kernels of csrc/gg_controller.cu through the C ABI (include/greengate_b200.h):

  AdmissionController.decide          -> gg_admit   (K1, n = 1)
  AdmissionController.decide_batch    -> gg_admit   (K1, frozen snapshot, n rows)
  AdmissionController.record_outcome  -> gg_outcome (K2, n = 1)
  AdmissionController.record_outcomes -> gg_outcome (K2, n outcomes in order)
  entropy_utility / one_minus_confidence_utility -> gg_utility
  threshold_at -> gg_threshold;  cost -> gg_cost

The controller state (normalizers, EWMA, latency window, counters) is one
`gg_state` struct in device memory (a torch uint8 tensor).  There is no CPU
fallback: without the library or a CUDA device, construction raises
`NativeUnavailable`.
"""

from __future__ import annotations

import contextlib
import ctypes as C
import math
import struct
import threading
import warnings
from dataclasses import dataclass, field, replace
from enum import Enum
from typing import Callable, Sequence

from . import _abi, _native
from .energy import EnergyLedger
from . import errors as _errors
from .errors import InvalidDistribution, InvalidSchedule, NegativeMeasurement, from_status


class Direction(Enum):
    GEQ = "GEQ"
    LT = "LT"

    def admits(self, composite: float, threshold: float) -> bool:
        """controller.py:44-47 (comparison only; used by the host API surface)."""
        if self is Direction.GEQ:
            return composite >= threshold
        return composite < threshold


class UtilityProxy(Enum):
    ENTROPY = "ENTROPY"
    ONE_MINUS_CONFIDENCE = "ONE_MINUS_CONFIDENCE"


class RoutePolicy(Enum):
    ALL_DIRECT = "ALL_DIRECT"
    ALL_BATCHED = "ALL_BATCHED"
    THRESHOLD_ON_QUEUE = "THRESHOLD_ON_QUEUE"


class ServicePath(Enum):
    DIRECT = "DIRECT"
    BATCHED = "BATCHED"
    NONE = "NONE"


class Reason(Enum):
    ADMITTED = "ADMITTED"
    BELOW_THRESHOLD = "BELOW_THRESHOLD"
    ABOVE_THRESHOLD = "ABOVE_THRESHOLD"


_DIR = {Direction.GEQ: _abi.GG_DIR_GEQ, Direction.LT: _abi.GG_DIR_LT}
_UTIL = {UtilityProxy.ENTROPY: _abi.GG_UTIL_ENTROPY,
         UtilityProxy.ONE_MINUS_CONFIDENCE: _abi.GG_UTIL_ONE_MINUS_CONFIDENCE}
_ROUTE = {RoutePolicy.ALL_DIRECT: _abi.GG_ROUTE_ALL_DIRECT,
          RoutePolicy.ALL_BATCHED: _abi.GG_ROUTE_ALL_BATCHED,
          RoutePolicy.THRESHOLD_ON_QUEUE: _abi.GG_ROUTE_THRESHOLD_ON_QUEUE}
_PATH_OF_CODE = {_abi.GG_DECISION_SKIP: ServicePath.NONE,
                 _abi.GG_DECISION_DIRECT: ServicePath.DIRECT,
                 _abi.GG_DECISION_BATCHED: ServicePath.BATCHED}


def _enum(cls, v):
    """Accept the reference's enum members (or names) as well as ours."""
    if isinstance(v, cls):
        return v
    return cls[getattr(v, "name", v)]


@dataclass(frozen=True)
class CostWeights:
    alpha: float
    beta: float
    gamma: float

    def __post_init__(self) -> None:
        for name in ("alpha", "beta", "gamma"):
            if not math.isfinite(getattr(self, name)):
                raise ValueError(f"weight {name} must be finite")


@dataclass(frozen=True)
class ThresholdSchedule:
    tau0: float
    tau_inf: float
    k: float
    t_origin: float = 0.0

    def __post_init__(self) -> None:
        fields = (self.tau0, self.tau_inf, self.k, self.t_origin)
        if not all(math.isfinite(v) for v in fields):
            raise InvalidSchedule(f"schedule fields must be finite, got {self}")
        if self.k <= 0.0:
            raise InvalidSchedule(f"decay rate k must be > 0, got {self.k!r}")
        if self.tau0 < self.tau_inf:
            warnings.warn("threshold schedule rises over time (tau0 < tau_inf); "
                          "decay-from-permissive runs expect tau0 >= tau_inf", stacklevel=2)


@dataclass(frozen=True)
class CostBreakdown:
    utility: float
    energy: float
    congestion: float
    composite: float
    threshold: float


@dataclass(frozen=True)
class AdmissionDecision:
    admit: bool
    path: ServicePath
    breakdown: CostBreakdown
    reason: Reason


@dataclass
class NormalizerChannel:
    """Host view of one device normalizer channel (controller.py:157-183)."""

    running_min: float | None = None
    running_max: float | None = None

    def observe(self, raw: float) -> None:
        if self.running_min is None or raw < self.running_min:
            self.running_min = raw
        if self.running_max is None or raw > self.running_max:
            self.running_max = raw

    def normalize(self, raw: float) -> float:
        self.observe(raw)
        lo, hi = self.running_min, self.running_max
        if hi <= lo:
            return 0.0
        return min(1.0, max(0.0, (raw - lo) / (hi - lo)))

    def copy(self) -> "NormalizerChannel":
        return NormalizerChannel(self.running_min, self.running_max)


@dataclass
class NormalizerState:
    energy: NormalizerChannel = field(default_factory=NormalizerChannel)
    queue_depth: NormalizerChannel = field(default_factory=NormalizerChannel)
    p95_ms: NormalizerChannel = field(default_factory=NormalizerChannel)


@dataclass(frozen=True)
class CongestionSnapshot:
    """servesim.py:113-119."""

    queue_depth: int
    p95_latency_ms: float
    batch_fill: float


# --------------------------------------------------------------- device helpers

class _Device:
    """Per-process scratch buffers for the stateless helpers (one per device).

    `use()` holds the lock across the whole copy -> launch -> read-back
    sequence, so concurrent callers (threads, or different current streams)
    never see each other's inputs; the reference functions are pure and
    thread-safe, and so are these."""

    _lock = threading.RLock()
    _scratch: dict = {}

    @classmethod
    def _tensors(cls, device, n: int, k: int):
        torch = _native.require_cuda()
        key = (str(device),)
        buf = cls._scratch.get(key)
        if buf is None or buf["cap"] < n * max(k, 3):
            cap = max(64, n * max(k, 3))
            buf = {"cap": cap,
                   "in": torch.empty(cap, dtype=torch.float64, device=device),
                   "out": torch.empty(cap, dtype=torch.float64, device=device),
                   "valid": torch.empty(cap, dtype=torch.uint8, device=device)}
            cls._scratch[key] = buf
        return buf

    @classmethod
    @contextlib.contextmanager
    def use(cls, device, n: int, k: int):
        with cls._lock:
            yield cls._tensors(device, n, k)


def _default_device():
    torch = _native.require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


def _utility_device(scores: Sequence[float], proxy: UtilityProxy) -> float:
    torch = _native.require_cuda()
    lib = _native.load()
    xs = [float(s) for s in scores]
    if len(xs) < 2:
        raise InvalidDistribution(f"need at least 2 class scores, got {len(xs)}")
    dev = _default_device()
    host = torch.tensor(xs, dtype=torch.float64)
    with _Device.use(dev, 1, len(xs)) as buf:
        buf["in"][: len(xs)].copy_(host)
        _native.check("gg_utility", lib.gg_utility(_native.ptr(buf["in"]), 1, len(xs), len(xs),
                                                   _UTIL[proxy], _native.ptr(buf["out"]),
                                                   _native.ptr(buf["valid"]), _native.stream_ptr()))
        u = float(buf["out"][0].item())
        valid = int(buf["valid"][0].item())
    if not valid:
        total = sum(xs)
        if any(not math.isfinite(x) or x < 0.0 for x in xs):
            raise InvalidDistribution(f"scores must be finite and >= 0: {xs}")
        raise InvalidDistribution(f"scores must sum to 1 (got {total!r})")
    return u


def entropy_utility(scores: Sequence[float]) -> float:
    """controller.py:138-142, evaluated by the device (gg_utility)."""
    return _utility_device(scores, UtilityProxy.ENTROPY)


def one_minus_confidence_utility(scores: Sequence[float]) -> float:
    """controller.py:145-148, evaluated by the device (gg_utility)."""
    return _utility_device(scores, UtilityProxy.ONE_MINUS_CONFIDENCE)


def threshold_at(schedule: ThresholdSchedule, t: float) -> float:
    """controller.py:114-123, evaluated by the device (gg_threshold)."""
    if not (math.isfinite(schedule.k) and schedule.k > 0.0):
        raise InvalidSchedule(f"decay rate k must be > 0, got {schedule.k!r}")
    lib = _native.load()
    with _Device.use(_default_device(), 1, 1) as buf:
        buf["in"][:1].fill_(float(t))
        _native.check("gg_threshold", lib.gg_threshold(schedule.tau0, schedule.tau_inf, schedule.k,
                                                       schedule.t_origin, _native.ptr(buf["in"]),
                                                       _native.ptr(buf["out"]), 1,
                                                       _native.stream_ptr()))
        return float(buf["out"][0].item())


def cost(weights: CostWeights, utility: float, energy: float, congestion: float) -> float:
    """controller.py:214-216, evaluated by the device (gg_cost)."""
    lib = _native.load()
    torch = _native.require_cuda()
    host = torch.tensor([utility, energy, congestion], dtype=torch.float64)
    with _Device.use(_default_device(), 1, 3) as buf:
        buf["in"][:3].copy_(host)
        _native.check("gg_cost", lib.gg_cost(weights.alpha, weights.beta, weights.gamma,
                                             _native.ptr(buf["in"]), _native.ptr(buf["out"]), 1,
                                             _native.stream_ptr()))
        return float(buf["out"][0].item())


_UTILITY_FN = {UtilityProxy.ENTROPY: entropy_utility,
               UtilityProxy.ONE_MINUS_CONFIDENCE: one_minus_confidence_utility}


# ------------------------------------------------------------------ config

@dataclass(frozen=True)
class ControllerConfig:
    """controller.py:219-253; `build` returns the device-backed controller."""

    enabled: bool = True
    alpha: float = 1.0
    beta: float = 0.0
    gamma: float = 0.0
    tau0: float = 1.0
    tau_inf: float = 0.2
    k: float = 0.5
    direction: Direction = Direction.GEQ
    utility_proxy: UtilityProxy = UtilityProxy.ENTROPY
    routing: RoutePolicy = RoutePolicy.ALL_DIRECT
    queue_threshold: int = 4

    def build(self, ledger=None, congestion_source=None, *, p95_window: int = 100,
              t_origin: float = 0.0, device=None) -> "AdmissionController":
        ctl = AdmissionController(
            CostWeights(self.alpha, self.beta, self.gamma),
            ThresholdSchedule(self.tau0, self.tau_inf, self.k, t_origin),
            ledger if ledger is not None else EnergyLedger(),
            congestion_source,
            direction=_enum(Direction, self.direction),
            utility_proxy=_enum(UtilityProxy, self.utility_proxy),
            routing=_enum(RoutePolicy, self.routing),
            queue_threshold=self.queue_threshold,
            p95_window=p95_window,
            device=device,
        )
        # `enabled` is read by the serving loop, as the reference's simulator reads it
        # (servesim.py:231-240): GatedServer(open_loop=None) runs the open-loop arm
        # for a controller built from a disabled config
        ctl.enabled = bool(self.enabled)
        return ctl


@dataclass
class BatchDecision:
    """Device-resident result of `decide_batch` (K1 over a micro-batch).

    decision      u8[n]  GG_DECISION_* (0 skip, 1 direct, 2 batched, 255 invalid)
    breakdown     f64[n, 3] (utility, composite, threshold) or None
    admitted_idx  i32[n]; the first `n_admitted` entries are the admitted rows, ascending
    info          u8[48] gg_batch_info (n_admitted, n_skipped, n_invalid, first_invalid, E, C)
    """

    decision: object
    breakdown: object
    admitted_idx: object
    info: object

    def summary(self) -> dict:
        raw = bytes(self.info.cpu().numpy().tobytes())
        b = _abi.gg_batch_info.from_buffer_copy(raw)
        return {"n_admitted": b.n_admitted, "n_skipped": b.n_skipped, "n_invalid": b.n_invalid,
                "first_invalid": b.first_invalid, "energy": b.energy, "congestion": b.congestion}

    @property
    def n_admitted(self) -> int:
        return int(self.summary()["n_admitted"])

    def admitted(self):
        return self.admitted_idx[: self.n_admitted]


class AdmissionController:
    """Per-request admit/skip policy driven by measured outcomes (controller.py:256-362).

    All mutations are stream-ordered on the CUDA stream current at call time;
    like the reference, the object holds no lock — callers serialize.
    """

    def __init__(self, weights: CostWeights, schedule: ThresholdSchedule, ledger,
                 congestion_source: Callable[[], object] | None = None, *,
                 direction: Direction = Direction.GEQ,
                 utility_proxy: UtilityProxy = UtilityProxy.ENTROPY,
                 routing: RoutePolicy = RoutePolicy.ALL_DIRECT, queue_threshold: int = 4,
                 p95_window: int = 100, device=None) -> None:
        torch = _native.require_cuda()
        self._lib = _native.load()
        self.device = torch.device(device) if device is not None else _default_device()
        # Ledgers of the reference package (or any foreign object) are mirrored:
        # the device owns the EWMA, the foreign object's fields are refreshed
        # after each outcome so callers that read it keep seeing current values.
        if isinstance(ledger, EnergyLedger):
            self.ledger, self._mirror = ledger, None
        else:
            self.ledger = EnergyLedger(grid_intensity=ledger.grid_intensity,
                                       ewma_lambda=ledger.ewma_lambda,
                                       total_joules=ledger.total_joules,
                                       ewma_joules_per_request=ledger.ewma_joules_per_request,
                                       samples_seen=ledger.samples_seen)
            self._mirror = ledger
        # exception classes raised by decide()/record_outcome(): ours, or (when
        # patched into a host package, integration.py) classes deriving from
        # both the host's and ours, so either side's `except` clauses match
        self.errors = _errors
        # policy attributes: assigning any of them (like the reference, whose
        # decide() reads them on every call) rebuilds the device parameter block
        self._policy = dict(weights=weights, schedule=schedule,
                            direction=_enum(Direction, direction),
                            utility_proxy=_enum(UtilityProxy, utility_proxy),
                            routing=_enum(RoutePolicy, routing),
                            queue_threshold=int(queue_threshold))
        self.congestion_source = congestion_source
        self.p95_window = int(p95_window)
        self.params = self._build_params(self._policy)
        with torch.cuda.device(self.device):
            self.state = torch.zeros(_abi.STATE_BYTES, dtype=torch.uint8, device=self.device)
            self._ws = torch.zeros(self._lib.gg_admit_workspace_bytes(1), dtype=torch.uint8,
                                   device=self.device)
            # single-call staging: one H2D of packed inputs, one D2H of packed outputs
            self._io = torch.empty(0, dtype=torch.uint8, device=self.device)
            self._io_k = -1
            self._snap_dev = torch.zeros(_abi.SNAPSHOT_BYTES, dtype=torch.uint8, device=self.device)
            self._err = torch.empty(1, dtype=torch.int64, device=self.device)
            st = self._stream()
            _native.check("gg_state_init", self._lib.gg_state_init(
                _native.ptr(self.state), schedule.t_origin, st))
            self._seed_from_ledger()
        self.ledger._bind(self)
        import sys
        self.result_types = sys.modules[__name__]

    # ------------------------------------------------------------------ plumbing
    def _build_params(self, pol: dict) -> _abi.gg_params:
        w, sc = pol["weights"], pol["schedule"]
        p = _abi.gg_params(
            w.alpha, w.beta, w.gamma, sc.tau0, sc.tau_inf, sc.k, self.ledger.ewma_lambda,
            _DIR[_enum(Direction, pol["direction"])],
            _UTIL[_enum(UtilityProxy, pol["utility_proxy"])],
            _ROUTE[_enum(RoutePolicy, pol["routing"])], int(pol["queue_threshold"]),
            self.p95_window, 0)
        rc = self._lib.gg_validate_params(C.byref(p))
        if rc != _abi.GG_OK:
            raise from_status(rc, f"invalid controller parameters (gg_status {rc})")
        return p

    def _set_policy(self, name: str, value) -> None:
        pol = dict(self._policy)
        pol[name] = value
        self.params = self._build_params(pol)   # validates before committing
        self._policy = pol

    def _stream(self):
        torch = _native.require_cuda()
        return _native.stream_ptr(torch.cuda.current_stream(self.device))

    def _seed_from_ledger(self) -> None:
        """Carry a pre-used ledger's EWMA into the device state (build() with a
        ledger that has already seen samples)."""
        led = self.ledger
        if led._seen == 0 and led._total == 0.0:
            return
        torch = _native.require_cuda()
        host = self.state.cpu()
        s = _abi.gg_state.from_buffer(bytearray(host.numpy().tobytes()))
        s.ewma_joules_per_request = led._ewma
        s.samples_seen = led._seen
        s.total_joules = led._total
        s.t_origin = self.schedule.t_origin
        self.state.copy_(torch.frombuffer(bytearray(bytes(s)), dtype=torch.uint8))

    def _state_scalar(self, name: str):
        off = _abi.STATE_OFFSETS[name]
        ctype = dict(_abi.gg_state._fields_)[name]
        size = C.sizeof(ctype)
        raw = bytes(self.state[off: off + size].cpu().numpy().tobytes())
        return ctype.from_buffer_copy(raw).value

    def state_struct(self) -> _abi.gg_state:
        """Copy of the full device state as a gg_state ctypes struct."""
        return _abi.gg_state.from_buffer_copy(bytes(self.state.cpu().numpy().tobytes()))

    def _ensure_ws(self, n: int) -> None:
        need = self._lib.gg_admit_workspace_bytes(int(n))
        if self._ws.numel() < need:
            torch = _native.require_cuda()
            self._ws = torch.zeros(need, dtype=torch.uint8, device=self.device)

    def _sync_mirror(self) -> None:
        m = self._mirror
        if m is None:
            return
        s = self.state_struct()
        m.ewma_joules_per_request = s.ewma_joules_per_request
        m.samples_seen = s.samples_seen
        m.total_joules = s.total_joules + self.ledger._extra

    # ------------------------------------------------------------------ reference API
    @property
    def schedule(self) -> ThresholdSchedule:
        return self._policy["schedule"]

    @schedule.setter
    def schedule(self, value: ThresholdSchedule) -> None:
        """A replacement schedule takes effect on the next decide(): tau0 /
        tau_inf / k go into the parameter block, t_origin into the device state."""
        self._set_policy("schedule", value)
        _native.check("gg_reset_clock", self._lib.gg_reset_clock(
            _native.ptr(self.state), value.t_origin, self._stream()))

    @property
    def weights(self) -> CostWeights:
        return self._policy["weights"]

    @weights.setter
    def weights(self, value: CostWeights) -> None:
        self._set_policy("weights", value)

    @property
    def direction(self) -> Direction:
        return self._policy["direction"]

    @direction.setter
    def direction(self, value) -> None:
        self._set_policy("direction", _enum(Direction, value))

    @property
    def utility_proxy(self) -> UtilityProxy:
        return self._policy["utility_proxy"]

    @utility_proxy.setter
    def utility_proxy(self, value) -> None:
        self._set_policy("utility_proxy", _enum(UtilityProxy, value))

    @property
    def routing(self) -> RoutePolicy:
        return self._policy["routing"]

    @routing.setter
    def routing(self, value) -> None:
        self._set_policy("routing", _enum(RoutePolicy, value))

    @property
    def queue_threshold(self) -> int:
        return self._policy["queue_threshold"]

    @queue_threshold.setter
    def queue_threshold(self, value: int) -> None:
        self._set_policy("queue_threshold", int(value))

    @property
    def admitted_total(self) -> int:
        return int(self._state_scalar("admitted_total"))

    @property
    def skipped_total(self) -> int:
        return int(self._state_scalar("skipped_total"))

    @property
    def normalizers(self) -> NormalizerState:
        s = self.state_struct()

        def ch(c):
            return NormalizerChannel(c.lo, c.hi) if c.seen else NormalizerChannel()
        return NormalizerState(ch(s.n_energy), ch(s.n_queue_depth), ch(s.n_p95_ms))

    def p95_ms(self) -> float:
        """controller.py:289-293 (maintained on device by K2)."""
        return float(self._state_scalar("p95_current"))

    def _snapshot_struct(self):
        if self.congestion_source is None:
            return None
        snap = self.congestion_source()
        return _abi.gg_snapshot(int(snap.queue_depth), float(snap.p95_latency_ms),
                                float(snap.batch_fill))

    # single-call io buffer layout (bytes): [scores f64 x k | now f64 | snapshot 24 |
    # breakdown 3 x f64 | batch_info 48 | decision u8 (+7 pad)]
    def _io_buffer(self, k: int):
        if self._io_k != k:
            torch = _native.require_cuda()
            self._io = torch.empty(8 * (k + 1) + 24 + 24 + _abi.BATCH_INFO_BYTES + 8,
                                   dtype=torch.uint8, device=self.device)
            self._io_k = k
        return self._io

    def decide(self, features, now: float) -> AdmissionDecision:
        """controller.py:309-343: one H2D, one K1 launch (n = 1), one D2H."""
        torch = _native.require_cuda()
        xs = [float(s) for s in features.scores]
        k = len(xs)
        E = self.errors
        if k < 2:
            raise E.InvalidDistribution(f"need at least 2 class scores, got {k}")
        snap = self._snapshot_struct()
        io = self._io_buffer(k)
        o_snap = 8 * (k + 1)
        o_out = o_snap + 24
        packed = struct.pack(f"<{k + 1}d", *xs, float(now)) + (bytes(snap) if snap else bytes(24))
        io[:o_out].copy_(torch.frombuffer(bytearray(packed), dtype=torch.uint8))
        base = io.data_ptr()
        _native.check("gg_admit", self._lib.gg_admit(
            C.byref(self.params), _native.ptr(self.state), C.c_void_p(base), 1, k, k,
            C.c_void_p(base + 8 * k), C.c_void_p(base + o_snap) if snap is not None else None,
            C.c_void_p(base + o_out + 24 + _abi.BATCH_INFO_BYTES), C.c_void_p(base + o_out), None,
            C.c_void_p(base + o_out + 24), _native.ptr(self._ws), self._ws.numel(),
            self._stream()))
        raw = bytes(io[o_out:].cpu().numpy().tobytes())
        bd = struct.unpack_from("<3d", raw, 0)
        info = _abi.gg_batch_info.from_buffer_copy(raw, 24)
        code = raw[24 + _abi.BATCH_INFO_BYTES]
        if code == _abi.GG_DECISION_INVALID:
            if any(not math.isfinite(x) or x < 0.0 for x in xs):
                raise E.InvalidDistribution(f"scores must be finite and >= 0: {xs}")
            raise E.InvalidDistribution(f"scores must sum to 1 (got {sum(xs)!r})")
        admit = code in (_abi.GG_DECISION_DIRECT, _abi.GG_DECISION_BATCHED)
        # result types: ours, or the host package's when patched into it (integration.py)
        T = self.result_types
        if admit:
            reason = T.Reason.ADMITTED
        else:
            reason = (T.Reason.BELOW_THRESHOLD if self.direction is Direction.GEQ
                      else T.Reason.ABOVE_THRESHOLD)
        return T.AdmissionDecision(admit=admit, path=T.ServicePath[_PATH_OF_CODE[code].name],
                                   breakdown=T.CostBreakdown(bd[0], info.energy, info.congestion,
                                                             bd[1], bd[2]),
                                   reason=reason)

    def record_outcome(self, latency_ms: float, joules: float, queue_depth: int) -> None:
        """controller.py:345-358: one K2 launch (stream-ordered, no host sync)."""
        if latency_ms < 0.0 or joules < 0.0 or queue_depth < 0:
            raise self.errors.NegativeMeasurement(
                f"outcome measurements must be >= 0, got "
                f"latency={latency_ms!r} joules={joules!r} depth={queue_depth!r}")
        torch = _native.require_cuda()
        io = self._io_buffer(max(self._io_k, 2))
        io[:24].copy_(torch.frombuffer(
            bytearray(struct.pack("<ddi4x", float(latency_ms), float(joules), int(queue_depth))),
            dtype=torch.uint8))
        base = io.data_ptr()
        _native.check("gg_outcome", self._lib.gg_outcome(
            C.byref(self.params), _native.ptr(self.state), C.c_void_p(base), C.c_void_p(base + 8),
            C.c_void_p(base + 16), 1, 0, None, self._stream()))
        if self._mirror is not None:
            self._sync_mirror()

    def reset_clock(self, t_origin: float) -> None:
        """controller.py:360-362."""
        self.schedule = replace(self.schedule, t_origin=t_origin)

    # ------------------------------------------------------------------ batch API
    def decide_batch(self, scores, now, snapshot=None, *, breakdown: bool = True,
                     out: BatchDecision | None = None) -> BatchDecision:
        """K1 over a micro-batch against one frozen snapshot.

        scores: CUDA f64 [n, k] (row stride may exceed k); now: CUDA f64 [n].
        snapshot: None (congestion_source, or the default snapshot), a
        CongestionSnapshot-like object, or a CUDA uint8 tensor holding a
        gg_snapshot (device-resident, e.g. written by the serving loop).
        Equivalent to calling decide() on every row in order with that
        snapshot; invalid rows get code 255 and change no state.
        """
        torch = _native.require_cuda()
        if scores.dim() != 2:
            raise ValueError(f"scores must be [n, k], got shape {tuple(scores.shape)}")
        n, k = int(scores.shape[0]), int(scores.shape[1])
        if scores.dtype != torch.float64 or now.dtype != torch.float64:
            raise TypeError("scores and now must be float64 CUDA tensors")
        self._check_device(scores=scores, now=now)
        if n > 0 and k > 1 and scores.stride(1) != 1:
            raise ValueError("scores rows must be contiguous")
        if now.dim() != 1 or now.numel() < n or (n > 0 and now.stride(0) != 1):
            raise ValueError(f"now must be a contiguous [n] tensor with n >= {n}, "
                             f"got shape {tuple(now.shape)}")
        self._ensure_ws(n)
        if out is None:
            out = BatchDecision(
                decision=torch.empty(n, dtype=torch.uint8, device=self.device),
                breakdown=torch.empty((n, 3), dtype=torch.float64, device=self.device) if breakdown else None,
                admitted_idx=torch.empty(max(n, 1), dtype=torch.int32, device=self.device),
                info=torch.empty(_abi.BATCH_INFO_BYTES, dtype=torch.uint8, device=self.device))
        snap_ptr = None
        if snapshot is None and self.congestion_source is not None:
            snapshot = self.congestion_source()
        if snapshot is not None:
            if hasattr(snapshot, "data_ptr"):
                snap_ptr = _native.ptr(snapshot)
            else:
                s = _abi.gg_snapshot(int(snapshot.queue_depth), float(snapshot.p95_latency_ms),
                                     float(snapshot.batch_fill))
                self._snap_dev.copy_(torch.frombuffer(bytearray(bytes(s)), dtype=torch.uint8))
                snap_ptr = _native.ptr(self._snap_dev)
        _native.check("gg_admit", self._lib.gg_admit(
            C.byref(self.params), _native.ptr(self.state), _native.ptr(scores), n, k,
            max(k, int(scores.stride(0))), _native.ptr(now), snap_ptr, _native.ptr(out.decision),
            _native.ptr(out.breakdown), _native.ptr(out.admitted_idx), _native.ptr(out.info),
            _native.ptr(self._ws), self._ws.numel(), self._stream()))
        return out

    def record_outcomes(self, latency_ms, joules, queue_depth, *, set_queue_depth: bool = False,
                        check: bool = True):
        """K2 over n served requests in completion order (CUDA f64, f64, i32 tensors).

        Returns the device int64 error index (-1 == all applied).  With
        check=True the call syncs and raises NegativeMeasurement like a Python
        loop over record_outcome would (outcomes before the bad one stay applied).
        """
        torch = _native.require_cuda()
        for name, t, dt in (("latency_ms", latency_ms, torch.float64),
                            ("joules", joules, torch.float64),
                            ("queue_depth", queue_depth, torch.int32)):
            if not hasattr(t, "data_ptr") or t.dtype != dt:
                raise TypeError(f"{name} must be a {dt} CUDA tensor, got "
                                f"{getattr(t, 'dtype', type(t).__name__)}")
            if t.dim() != 1 or (t.numel() > 1 and t.stride(0) != 1):
                raise ValueError(f"{name} must be a contiguous 1-D tensor")
        self._check_device(latency_ms=latency_ms, joules=joules, queue_depth=queue_depth)
        n = int(latency_ms.shape[0])
        if int(joules.shape[0]) != n or int(queue_depth.shape[0]) != n:
            raise ValueError(f"latency_ms, joules and queue_depth must have equal lengths, got "
                             f"{n}, {int(joules.shape[0])}, {int(queue_depth.shape[0])}")
        _native.check("gg_outcome", self._lib.gg_outcome(
            C.byref(self.params), _native.ptr(self.state), _native.ptr(latency_ms),
            _native.ptr(joules), _native.ptr(queue_depth), n, int(set_queue_depth),
            _native.ptr(self._err), self._stream()))
        if check:
            bad = int(self._err.item())
            if bad >= 0:
                raise self.errors.NegativeMeasurement(
                    f"outcome measurements must be >= 0, got latency={float(latency_ms[bad])!r} "
                    f"joules={float(joules[bad])!r} depth={int(queue_depth[bad])!r}")
            if self._mirror is not None:
                self._sync_mirror()
        return self._err

    def _check_device(self, **tensors) -> None:
        for name, t in tensors.items():
            if t.device != self.device:
                raise ValueError(f"{name} is on {t.device}, the controller on {self.device}")

    def set_queue_depth(self, depth: int) -> None:
        """The gateway's reported depth (gateway.py:191-192, 230) for the default snapshot."""
        _native.check("gg_set_queue_depth", self._lib.gg_set_queue_depth(
            _native.ptr(self.state), int(depth), self._stream()))
