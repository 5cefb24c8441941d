"""Gateway micro-batching front end.

The reference gateway (gateway.py:179-230) serializes every ``POST /v1/decide``
and ``POST /v1/outcome`` through one lock: one ``decide`` / ``record_outcome``
call per HTTP request, each against the state every earlier request left.
`GatewayBatcher` keeps exactly that contract — requests take a total order
(enqueue order), each is decided against the state of all earlier ones — but
drains the requests that queued up concurrently in one go:

* every maximal run of consecutive decides with the same score count and the
  same reported queue depth is ONE K1 launch (`AdmissionController.decide_batch`,
  frozen snapshot = the ``CongestionSnapshot(depth, p95, 0.0)`` the reference's
  ``GatewayState._congestion`` would build for each of them: nothing between
  them changes depth or p95);
* every run of consecutive valid outcomes is ONE K2 launch
  (`record_outcomes`, completion order); a negative measurement is rejected
  host-side (HTTP 400, no state change, depth not updated) exactly as
  ``record_outcome`` raising inside the reference's lock.

Request bodies, field validation, status codes and the JSON answer of
``/v1/decide`` follow the reference handler (`_field`, ``_ApiError`` → `ApiError`).
``now`` is the request's ``timestamp_s`` or ``clock()`` sampled at enqueue, in
enqueue order (the reference samples it under the lock, i.e. in lock order).
The HTTP server itself is out of scope; `decide` / `outcome` /
`reset` are what its handlers call.
"""

from __future__ import annotations

import math
import threading
import time
from concurrent.futures import Future
from dataclasses import dataclass
from typing import Any

from . import _abi
from .controller import ControllerConfig, CongestionSnapshot, Direction, _PATH_OF_CODE
from .energy import DEFAULT_EWMA_LAMBDA, EnergyLedger


class ApiError(Exception):
    """HTTP status + message, as the reference's ``_ApiError`` (gateway.py)."""

    def __init__(self, status: int, message: str) -> None:
        super().__init__(message)
        self.status = status
        self.message = message


def _field(body: dict, name: str, types: tuple, required: bool = True):
    """gateway.py:101-109: missing -> 422, wrong type (bools never match) -> 422."""
    if name not in body:
        if required:
            raise ApiError(422, f"missing field {name!r}")
        return None
    v = body[name]
    if isinstance(v, bool) or not isinstance(v, types):
        raise ApiError(422, f"field {name!r} has wrong type")
    return v


def _to_device(t, dev):
    """Host tensor -> the controller's device (pinned staging for CUDA)."""
    import torch
    dev = torch.device(dev)
    if dev.type != "cuda":
        return t
    return t.pin_memory().to(dev, non_blocking=True)


@dataclass
class _Item:
    kind: str                 # "decide" | "outcome" | "reset" | "barrier"
    fut: Future
    scores: tuple = ()
    now: float = 0.0
    depth: int | None = None
    latency_ms: float = 0.0
    joules: float = 0.0


class GatewayBatcher:
    """The reference ``GatewayState`` + handlers, with requests coalesced into
    batched K1 / K2 launches.  Thread-safe; `decide` / `outcome` block until
    their request has been applied."""

    def __init__(self, config: ControllerConfig | None, *, ewma_lambda: float = DEFAULT_EWMA_LAMBDA,
                 clock=time.monotonic, max_batch: int = 1024, max_wait_s: float = 200e-6,
                 device=None, controller=None, record_order: bool = False) -> None:
        self.clock = clock
        # record_order: keep (kind, body) in enqueue order — the total order the
        # answers are defined by (tests replay it through the sequential gateway)
        self.order: list | None = [] if record_order else None
        self.queue_depth = 0
        self.max_batch = int(max_batch)
        self.max_wait_s = float(max_wait_s)
        if controller is not None:
            self.controller = controller
        elif config is not None:
            self.controller = config.build(EnergyLedger(ewma_lambda=ewma_lambda), self._congestion,
                                           t_origin=clock(), device=device)
        else:
            self.controller = None
        self.launches = {"decide": 0, "outcome": 0}   # K1 / K2 launches issued
        self._q: list[_Item] = []
        self._cv = threading.Condition()
        self._closed = False
        self._worker = threading.Thread(target=self._run, name="gg-gateway-batcher", daemon=True)
        self._worker.start()

    # ----------------------------------------------------------------- reference API
    def _congestion(self) -> CongestionSnapshot:
        """GatewayState._congestion: the last reported depth, the controller's p95."""
        return CongestionSnapshot(queue_depth=self.queue_depth,
                                  p95_latency_ms=self.controller.p95_ms(), batch_fill=0.0)

    def submit_decide(self, body: dict[str, Any]) -> Future:
        if self.controller is None:
            raise ApiError(503, "controller not configured")
        _field(body, "id", (str,))
        scores = _field(body, "scores", (list,))
        depth = _field(body, "queue_depth", (int,), required=False)
        ts = _field(body, "timestamp_s", (int, float), required=False)
        if not all(isinstance(s, (int, float)) and not isinstance(s, bool) for s in scores):
            raise ApiError(422, "field 'scores' must be an array of numbers")
        fut: Future = Future()
        with self._cv:
            if self._closed:
                raise ApiError(503, "gateway closed")
            now = float(ts) if ts is not None else self.clock()
            self._q.append(_Item("decide", fut, tuple(float(s) for s in scores), now, depth))
            if self.order is not None:
                self.order.append(("decide", body))
            self._cv.notify()
        return fut

    def submit_outcome(self, body: dict[str, Any]) -> Future:
        if self.controller is None:
            raise ApiError(503, "controller not configured")
        _field(body, "id", (str,))
        latency = float(_field(body, "latency_ms", (int, float)))
        joules = float(_field(body, "joules", (int, float)))
        depth = _field(body, "queue_depth", (int,))
        fut: Future = Future()
        with self._cv:
            if self._closed:
                raise ApiError(503, "gateway closed")
            self._q.append(_Item("outcome", fut, depth=depth, latency_ms=latency, joules=joules))
            if self.order is not None:
                self.order.append(("outcome", body))
            self._cv.notify()
        return fut

    def decide(self, body: dict[str, Any]) -> dict[str, Any]:
        """POST /v1/decide (gateway.py:179-214)."""
        return self.submit_decide(body).result()

    def outcome(self, body: dict[str, Any]) -> None:
        """POST /v1/outcome (gateway.py:216-230)."""
        return self.submit_outcome(body).result()

    def submit_reset(self) -> Future:
        """POST /v1/reset (gateway.py:232-237): queued like any request, so the
        worker applies it in enqueue order (after every earlier request, before
        every later one) on its own stream; `now` is sampled at enqueue."""
        if self.controller is None:
            raise ApiError(503, "controller not configured")
        fut: Future = Future()
        with self._cv:
            if self._closed:
                raise ApiError(503, "gateway closed")
            now = self.clock()
            self._q.append(_Item("reset", fut, now=now))
            if self.order is not None:
                self.order.append(("reset", {"t_origin": now}))
            self._cv.notify()
        return fut

    def reset(self) -> None:
        """POST /v1/reset: re-arm the threshold clock (in request order)."""
        return self.submit_reset().result()

    def flush(self) -> None:
        """Block until every request queued before this call has been applied."""
        fut: Future = Future()
        with self._cv:
            if self._closed:
                raise ApiError(503, "gateway closed")
            self._q.append(_Item("barrier", fut))
            self._cv.notify()
        fut.result()

    def close(self) -> None:
        with self._cv:
            self._closed = True
            self._cv.notify()
        self._worker.join()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def _pinned(self, name: str, nbytes: int):
        """A reused pinned host buffer of >= nbytes (grown by doubling)."""
        import torch
        bufs = self.__dict__.setdefault("_pin", {})
        b = bufs.get(name)
        if b is None or b.numel() < nbytes:
            b = bufs[name] = torch.empty(max(nbytes, 2 * (b.numel() if b is not None else 0), 4096),
                                         dtype=torch.uint8).pin_memory()
        return b

    # ----------------------------------------------------------------- worker
    def _run(self) -> None:
        while True:
            with self._cv:
                while not self._q and not self._closed:
                    self._cv.wait()
                if not self._q and self._closed:
                    return
                deadline = time.monotonic() + self.max_wait_s
                while len(self._q) < self.max_batch and not self._closed:
                    rem = deadline - time.monotonic()
                    if rem <= 0:
                        break
                    self._cv.wait(rem)
                items, self._q = self._q[:self.max_batch], self._q[self.max_batch:]
            try:
                self._process(items)
            except BaseException as exc:   # never strand a caller
                for it in items:
                    if not it.fut.done():
                        it.fut.set_exception(exc)

    def _process(self, items: list[_Item]) -> None:
        i, n = 0, len(items)
        while i < n:
            it = items[i]
            if it.kind == "barrier":
                it.fut.set_result(None)
                i += 1
            elif it.kind == "reset":
                self.controller.reset_clock(it.now)
                it.fut.set_result(None)
                i += 1
            elif it.kind == "decide":
                # the run: consecutive decides, same k, same effective depth
                if it.depth is not None:
                    self.queue_depth = it.depth
                k, depth = len(it.scores), self.queue_depth
                j = i + 1
                while j < n and items[j].kind == "decide" and len(items[j].scores) == k and \
                        (items[j].depth is None or items[j].depth == depth):
                    j += 1
                self._decide_run(items[i:j], k, depth)
                i = j
            else:
                j = i
                while j < n and items[j].kind == "outcome":
                    j += 1
                self._outcome_run(items[i:j])
                i = j

    def _decide_run(self, run: list[_Item], k: int, depth: int) -> None:
        import torch
        ctl = self.controller
        if k < 2:   # decide() raises before touching the device (controller.py)
            for it in run:
                it.fut.set_exception(ApiError(400, f"need at least 2 class scores, got {k}"))
            return
        n = len(run)
        dev = torch.device(ctl.device)
        if dev.type == "cuda":
            # reused pinned staging: [scores n x k | now n] up, [codes | breakdown | info] down
            hin = self._pinned("in", n * (k + 1) * 8).view(torch.float64)
            hin[: n * k].view(n, k).copy_(torch.tensor([it.scores for it in run], dtype=torch.float64))
            hin[n * k: n * (k + 1)].copy_(torch.tensor([it.now for it in run], dtype=torch.float64))
            din = hin[: n * (k + 1)].to(dev, non_blocking=True)
            scores, now = din[: n * k].view(n, k), din[n * k:]
        else:
            scores = torch.tensor([it.scores for it in run], dtype=torch.float64)
            now = torch.tensor([it.now for it in run], dtype=torch.float64)
        snap = CongestionSnapshot(queue_depth=depth, p95_latency_ms=ctl.p95_ms(), batch_fill=0.0)
        out = ctl.decide_batch(scores, now, snap, breakdown=True)
        self.launches["decide"] += 1
        if dev.type == "cuda":
            hb = self._pinned("bd", n * 24).view(torch.float64)[: n * 3].view(n, 3)
            hc = self._pinned("dec", n)[:n]
            hi = self._pinned("info", _abi.BATCH_INFO_BYTES)[: _abi.BATCH_INFO_BYTES]
            hb.copy_(out.breakdown, non_blocking=True)
            hc.copy_(out.decision, non_blocking=True)
            hi.copy_(out.info, non_blocking=True)
            torch.cuda.current_stream(dev).synchronize()
            codes, bd = hc.tolist(), hb.tolist()
            info = _abi.gg_batch_info.from_buffer_copy(bytes(hi.numpy().tobytes()))
        else:
            codes = out.decision.tolist()
            bd = out.breakdown.tolist()
            info = _abi.gg_batch_info.from_buffer_copy(bytes(out.info.numpy().tobytes()))
        geq = ctl.direction is Direction.GEQ
        for it, code, (u, jv, tau) in zip(run, codes, bd):
            if code == _abi.GG_DECISION_INVALID:
                xs = it.scores
                msg = (f"scores must be finite and >= 0: {list(xs)}"
                       if any(not math.isfinite(x) or x < 0.0 for x in xs)
                       else f"scores must sum to 1 (got {sum(xs)!r})")
                it.fut.set_exception(ApiError(400, msg))
                continue
            admit = code in (_abi.GG_DECISION_DIRECT, _abi.GG_DECISION_BATCHED)
            reason = "ADMITTED" if admit else ("BELOW_THRESHOLD" if geq else "ABOVE_THRESHOLD")
            it.fut.set_result({"admit": admit, "path": _PATH_OF_CODE[code].name, "j": jv, "tau": tau,
                               "l": u, "e": info.energy, "c": info.congestion, "reason": reason})

    def _outcome_run(self, run: list[_Item]) -> None:
        import torch
        good = []
        for it in run:
            if it.latency_ms < 0.0 or it.joules < 0.0 or it.depth < 0:
                it.fut.set_exception(ApiError(
                    400, f"outcome measurements must be >= 0, got latency={it.latency_ms!r} "
                         f"joules={it.joules!r} depth={it.depth!r}"))
            else:
                good.append(it)
        if not good:
            return
        dev = self.controller.device
        lat = _to_device(torch.tensor([it.latency_ms for it in good], dtype=torch.float64), dev)
        jl = _to_device(torch.tensor([it.joules for it in good], dtype=torch.float64), dev)
        qd = _to_device(torch.tensor([it.depth for it in good], dtype=torch.int32), dev)
        self.controller.record_outcomes(lat, jl, qd, check=True)
        self.launches["outcome"] += 1
        self.queue_depth = good[-1].depth   # gateway.py:230, after the last applied outcome
        for it in good:
            it.fut.set_result(None)
