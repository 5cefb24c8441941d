"""Closed-loop gated serving on one GPU (optionally one of G data-parallel ranks).

One step, entirely on the device and captured as one CUDA graph:

  K1  gg_admit_stream     decide the next `window` trace rows against the
                          snapshot of the device FIFO (queue depth, p95, fill),
                          append the admitted rows to the FIFO ring in order
      gg_fifo_pop         pop up to B admitted requests -> batch ids + count
      gather              payloads of the served batch (images / token ids)
  fwd ResNet-18 / DistilBERT on the dynamic batch (count read on the device)
  K3  gg_epilogue_served  fp32 logits -> first-max prediction + fp64 confidence
      gg_served_outcomes  latency / joules / queue depth of the served batch
  K9  all_reduce(SUM)     rank-slotted outcome buffer (multi-GPU only; exact)
  K2  gg_outcome_slots    record_outcome() for every served request of every
                          rank, in rank order -> identical replicas

This replaces the reference's discrete-event stand-in for the serving backend
(pkg/src/greengate/servesim.py:280-367): admitted requests are queued and
served in fused batches (Path B, servesim.py:286-306), skipped ones are
answered by the zero-cost fallback and never reach the model.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

from . import _abi, _native

IMAGENET_MEAN = (0.485, 0.456, 0.406)
IMAGENET_STD = (0.229, 0.224, 0.225)


@dataclass
class OutcomeModel:
    """Latency/energy of a served batch (PathBConfig, servesim.py:62-71, 303-304).

    latency: "model"    base + per_item * n (service time only),
             "trace"    the reference's finish_t - enqueue_t in trace time:
                        queueing from arrival to the flush + the service time
                        (servesim.py:_maybe_flush, _complete),
             "measured" device %globaltimer from admission to completion.
    measured_latency=True is the older spelling of latency="measured"."""

    batch_base_ms: float = 4.0
    per_item_ms: float = 0.05
    batch_base_energy_j: float = 6.0
    per_item_energy_j: float = 1.5
    measured_latency: bool = False
    latency: str = "model"

    def mode(self) -> int:
        if self.measured_latency:
            return _abi.GG_LATENCY_MEASURED
        return {"model": _abi.GG_LATENCY_MODEL, "trace": _abi.GG_LATENCY_TRACE,
                "measured": _abi.GG_LATENCY_MEASURED}[self.latency]

    def abi(self) -> _abi.gg_outcome_model:
        return _abi.gg_outcome_model(self.batch_base_ms, self.per_item_ms,
                                     self.batch_base_energy_j, self.per_item_energy_j,
                                     self.mode(), 0)


class GatedServer:
    """Admission controller + device FIFO + forward pass + outcome feedback.

    controller: a device AdmissionController (paper_2601_04250_b200.controller)
    net:        ResNet18B200 or DistilBertB200 (its max_batch is B)
    scores/now: CUDA fp64 [T, K] / [T] resident trace (this rank's shard)
    payloads:   ResNet: CUDA uint8 [P, H, W, 3]; DistilBERT: (ids int32 [P, S], mask int32 [P, S])
    open_loop:  the reference's controller-disabled arm (servesim.py:231-240):
                admit every arrival, static route (gg_admit_open_stream); None
                follows the controller's config (`ControllerConfig.enabled`)
    batching_window_ms: Path-B flush policy (servesim.py:148-162): a batch is
                popped when B requests are pending or the oldest waited the
                window in trace time; None pops min(B, depth) every step
    labels / coins / fallback_degradation: fallback answers and accuracy
                accounting of every decided request (servesim.py:246-256);
                labels CUDA int32 [T], coins CUDA fp64 [>= T] (the `_fb_rng`
                stream, drawn on the host, see fallback_coins)
    pipeline:   software-pipelined steps (latency "model" or "trace"):
                the control chain of step t+1 (K1, fallback, pop, gather, served
                outcomes, K2) runs on the serving stream while step t's forward,
                K3 and publish run on a second stream.  No kernel of the control
                chain reads the forward's output, so every decision, answer,
                prediction and the controller state are the sequential loop's;
                the per-step buffers (batch ids / arrival stamps / count / batch
                info / model inputs / FIFO snapshot) alternate between two sets.
                run(n) completes n forwards with the control of the next step
                already done; flush() (or done() once the trace is served)
                completes the pending forward.
    """

    def __init__(self, controller, net, scores, now, payloads, *, window: int,
                 outcome: OutcomeModel | None = None, fifo_capacity: int = 1 << 20,
                 rank: int = 0, world: int = 1, process_group=None, open_loop: bool | None = None,
                 batching_window_ms: float | None = None, labels=None, coins=None,
                 fallback_degradation: float = 0.05, publish: bool = False,
                 pipeline: bool = False):
        torch = _native.require_cuda()
        self.torch = torch
        self.lib = _native.load()
        self.ctl, self.net = controller, net
        self.dev = controller.device
        self.B = int(net.max_batch)
        self.W = int(window)
        self.T, self.K = int(scores.shape[0]), int(scores.shape[1])
        self.scores, self.now = scores, now
        self.kind = "resnet18" if hasattr(net, "blocks") else "distilbert"
        self.payloads = payloads
        self.outcome_model = outcome or OutcomeModel()
        self.outcome = self.outcome_model.abi()
        self.rank, self.world, self.pg = rank, world, process_group
        if open_loop is None:
            open_loop = not getattr(controller, "enabled", True)
        self.open_loop = bool(open_loop)
        self.window_s = 0.0 if batching_window_ms is None else float(batching_window_ms) / 1000.0
        if self.window_s < 0.0:
            raise ValueError("batching_window_ms must be >= 0")
        self.trace_clock = batching_window_ms is not None or \
            self.outcome.measured_latency == _abi.GG_LATENCY_TRACE
        if (labels is None) != (coins is None):
            raise ValueError("labels and coins go together (fallback accounting)")
        if labels is not None:
            if labels.dtype != torch.int32 or coins.dtype != torch.float64:
                raise TypeError("labels must be int32 and coins float64 CUDA tensors")
            if labels.numel() < self.T or coins.numel() < self.T:
                raise ValueError("labels and coins need one entry per trace row")
        self.labels, self.coins = labels, coins
        self.fallback_degradation = float(fallback_degradation)
        assert fifo_capacity & (fifo_capacity - 1) == 0
        z = dict(device=self.dev)
        fifo = _abi.gg_fifo(0, 0, fifo_capacity, self.B, 0, self.T, 0, 0)
        self.fifo = torch.frombuffer(bytearray(bytes(fifo)), dtype=torch.uint8).to(self.dev)
        self.ring = torch.empty(fifo_capacity, dtype=torch.int32, **z)
        self.ring_ns = torch.empty(fifo_capacity, dtype=torch.int64, **z)
        self.pipeline = bool(pipeline)
        if self.pipeline and self.outcome.measured_latency == _abi.GG_LATENCY_MEASURED:
            raise ValueError("pipeline=True needs a latency model that does not time the "
                             "forward (latency='model' or 'trace')")
        self.batch_pred = torch.full((self.B,), -1, dtype=torch.int32, **z)
        self.batch_conf = torch.zeros(self.B, dtype=torch.float64, **z)
        self.slot_len = 3 * self.B + 8   # GG_SLOT_LEN(B)
        self.slots = torch.zeros(world * self.slot_len, dtype=torch.float64, **z)
        self.decision = torch.full((self.T,), 254, dtype=torch.uint8, **z)
        self.predicted = torch.full((self.T,), -1, dtype=torch.int32, **z)
        self.confidence = torch.full((self.T,), float("nan"), dtype=torch.float64, **z)
        # reference-semantics record columns (CompletionRecord, servesim.py:99-110)
        self.answer = torch.full((self.T,), -1, dtype=torch.int32, **z)       # predicted_label
        self.correct = torch.zeros(self.T, dtype=torch.uint8, **z)
        self.latency = torch.zeros(self.T, dtype=torch.float64, **z)        # latency_ms
        self.coin_cursor = torch.zeros(1, dtype=torch.int64, **z)
        self.ws = torch.zeros(self.lib.gg_admit_workspace_bytes(self.W), dtype=torch.uint8, **z)
        self.err = torch.empty(1, dtype=torch.int64, **z)
        if self.kind == "resnet18":
            self.mean = torch.tensor(IMAGENET_MEAN, dtype=torch.float32)
            self.std = torch.tensor(IMAGENET_STD, dtype=torch.float32)
        # per-step buffers: one set, or two alternating sets when pipelined
        self._sets = []
        for i in range(2 if self.pipeline else 1):
            d = dict(batch_ids=torch.full((self.B,), -1, dtype=torch.int32, **z),
                     batch_ns=torch.empty(self.B, dtype=torch.int64, **z),
                     count=torch.zeros(1, dtype=torch.int32, **z),
                     info=torch.empty(_abi.BATCH_INFO_BYTES, dtype=torch.uint8, **z),
                     fsnap=torch.empty_like(self.fifo) if self.pipeline else None)
            if self.kind == "resnet18":
                d["x16"] = net.x16 if i == 0 else torch.zeros_like(net.x16)   # zero borders
            else:
                d["tok_ids"] = torch.empty((self.B, net.seq_len), dtype=torch.int32, **z)
                d["tok_mask"] = torch.empty((self.B, net.seq_len), dtype=torch.int32, **z)
            self._sets.append(d)
        self._bind(0)
        self._ahead = False     # pipelined: the control of a step ran, its forward pending
        self._pset = 0          # pipelined: the set of that step
        self.control_steps = 0
        # publish: every step ends by writing its record (served predictions and
        # confidences, the window's decisions) into pinned host memory
        # (gg_publish_step), two slots alternating -- no device -> host copies
        self.publish = bool(publish)
        if self.publish:
            self.rec_bytes = int(self.lib.gg_step_record_bytes(self.B, self.W))
            self.host_records = torch.zeros(2 * self.rec_bytes, dtype=torch.uint8).pin_memory()
            self.rec_seq = torch.zeros(1, dtype=torch.int64, **z)
        self.graph = None
        self.stream = torch.cuda.Stream(device=self.dev)
        # Pipelined: the forward's persistent grids leave one TPC (2 SMs) free for the
        # control chain (gg_set_sm_reserve, applied to the captured graphs: it costs
        # the forward nothing at these tile counts), and one stream has the higher
        # priority -- the control stream for DistilBERT (its kernels are small and fit
        # the free TPC), the forward's for ResNet-18 (the image gather is a
        # 1792-block kernel that would take SMs from the forward).  Measured:
        # DESIGN.md section 7, finding I.
        import os
        self.sm_reserve = int(os.environ.get("GG_PIPE_SM_RESERVE", "2")) if self.pipeline else 0
        prio = os.environ.get("GG_PIPE_PRIO", "c" if self.kind == "distilbert" else "f")
        self.fstream = torch.cuda.Stream(device=self.dev, priority=-1 if prio == "f" else 0) \
            if self.pipeline else None
        if self.pipeline and prio == "c":
            self.stream = torch.cuda.Stream(device=self.dev, priority=-1)
        if self.pipeline:
            self._fork, self._join = torch.cuda.Event(), torch.cuda.Event()
        self.steps_run = 0

    def _bind(self, p: int) -> None:
        """Point the per-step buffer attributes at set p."""
        d = self._sets[p]
        self.batch_ids, self.batch_ns, self.count = d["batch_ids"], d["batch_ns"], d["count"]
        self.info, self._fsnap = d["info"], d["fsnap"]
        if self.kind == "resnet18":
            self._x16 = d["x16"]
        else:
            self.tok_ids, self.tok_mask = d["tok_ids"], d["tok_mask"]

    # ------------------------------------------------------------------ one step
    def _gather(self, st):
        """Payloads of the served batch -> this set's model inputs."""
        lib, B = self.lib, self.B
        if self.kind == "resnet18":
            pool = self.payloads
            H = int(pool.shape[1])
            _native.check("gg_stem_gather", lib.gg_stem_gather(
                _native.ptr(pool), int(pool.shape[0]), _native.ptr(self.batch_ids),
                _native.ptr(self.count), B, H, int(pool.shape[2]),
                self.mean.numpy().ctypes.data_as(C.c_void_p),
                self.std.numpy().ctypes.data_as(C.c_void_p), 1, _native.ptr(self._x16), st))
        else:
            ids, mask = self.payloads
            _native.check("gg_token_gather", lib.gg_token_gather(
                _native.ptr(ids), _native.ptr(mask), int(ids.shape[0]), _native.ptr(self.batch_ids),
                _native.ptr(self.count), B, self.net.seq_len, _native.ptr(self.tok_ids),
                _native.ptr(self.tok_mask), st))

    def _forward(self, st):
        B = self.B
        if self.kind == "resnet18":
            return self.net.forward_s2d(B, stream=self._cur_stream, count=self.count, x16=self._x16)
        return self.net.forward(self.tok_ids, self.tok_mask, batch=B, stream=self._cur_stream,
                                count=self.count)

    def step(self):
        """Enqueue one serving step on the current stream (graph-capturable)."""
        self.step_local()
        if self.world > 1:
            # K9: rank-slotted buffer, SUM == allgather exactly (x + 0 == x)
            self.torch.distributed.all_reduce(self.slots, group=self.pg)
        self.step_feedback()

    def step_local(self):
        """Admission, FIFO, forward, epilogue and this rank's exchange slot."""
        torch = self.torch
        self._cur_stream = torch.cuda.current_stream(self.dev)
        st = _native.stream_ptr(self._cur_stream)
        self._control_front(st)
        self._forward_tail(st)
        self._control_back(st)

    def _control_front(self, st):
        """K1 (decide the next window against the FIFO snapshot), fallback answers,
        the Path-B pop and the gather of the served batch's payloads."""
        lib, ctl = self.lib, self.ctl
        if self.open_loop:
            _native.check("gg_admit_open_stream", lib.gg_admit_open_stream(
                C.byref(ctl.params), _native.ptr(ctl.state), _native.ptr(self.fifo),
                _native.ptr(self.ring), _native.ptr(self.ring_ns), self.W,
                _native.ptr(self.decision), _native.ptr(self.info), st))
        else:
            _native.check("gg_admit_stream", lib.gg_admit_stream(
                C.byref(ctl.params), _native.ptr(ctl.state), _native.ptr(self.fifo),
                _native.ptr(self.ring), _native.ptr(self.ring_ns), _native.ptr(self.scores), self.K,
                int(self.scores.stride(0)), _native.ptr(self.now), self.W, None,
                _native.ptr(self.decision), _native.ptr(self.info), _native.ptr(self.ws),
                self.ws.numel(), st))
        if self.labels is not None:
            _native.check("gg_fallback_answers", lib.gg_fallback_answers(
                _native.ptr(self.scores), self.K, int(self.scores.stride(0)),
                _native.ptr(self.labels), _native.ptr(self.decision), _native.ptr(self.fifo),
                _native.ptr(self.info), 0, 0, _native.ptr(self.coins),
                _native.ptr(self.coin_cursor), self.fallback_degradation,
                _native.ptr(self.answer), _native.ptr(self.correct), st))
        if self.trace_clock:
            _native.check("gg_fifo_pop_windowed", lib.gg_fifo_pop_windowed(
                _native.ptr(self.fifo), _native.ptr(self.ring), _native.ptr(self.ring_ns),
                _native.ptr(self.now), self.window_s, _native.ptr(self.batch_ids),
                _native.ptr(self.batch_ns), _native.ptr(self.count), self.B, st))
        else:
            _native.check("gg_fifo_pop", lib.gg_fifo_pop(
                _native.ptr(self.fifo), _native.ptr(self.ring), _native.ptr(self.ring_ns),
                _native.ptr(self.batch_ids), _native.ptr(self.batch_ns), _native.ptr(self.count),
                self.B, st))
        if self._fsnap is not None:   # the window this step decided, for its publish
            self._fsnap.copy_(self.fifo, non_blocking=True)
        self._gather(st)

    def _forward_tail(self, st):
        """Forward on the gathered batch, K3 epilogue, publish of the step record."""
        lib = self.lib
        logits = self._forward(st)
        _native.check("gg_epilogue_served", lib.gg_epilogue_served(
            C.c_void_p(logits.data_ptr()), _native.ptr(self.count), self.B, int(logits.shape[1]),
            int(logits.stride(0)), _native.ptr(self.batch_ids), _native.ptr(self.predicted),
            _native.ptr(self.confidence), None, _native.ptr(self.batch_pred),
            _native.ptr(self.batch_conf), st))
        if self.publish:
            fifo = self._fsnap if self._fsnap is not None else self.fifo
            _native.check("gg_publish_step", lib.gg_publish_step(
                _native.ptr(self.count), _native.ptr(self.batch_pred), _native.ptr(self.batch_conf),
                _native.ptr(self.decision), _native.ptr(self.info), _native.ptr(fifo), self.B,
                self.W, C.c_void_p(self.host_records.data_ptr()), _native.ptr(self.rec_seq), st))

    def _control_back(self, st):
        """Served outcomes of the popped batch into this rank's exchange slot."""
        lib = self.lib
        if self.world > 1:
            self.slots.zero_()
        my_slot = self.slots[self.rank * self.slot_len:]
        _native.check("gg_served_outcomes_trace", lib.gg_served_outcomes_trace(
            _native.ptr(self.fifo), _native.ptr(self.count), _native.ptr(self.batch_ns),
            _native.ptr(self.batch_ids), _native.ptr(self.now), C.byref(self.outcome),
            _native.ptr(self.info), _native.ptr(my_slot), self.B, _native.ptr(self.latency), st))

    # ------------------------------------------------------------------ pipelined steps
    def _pipe_control(self, p, feedback: bool = True):
        """Control chain of one step into set p, on the current stream (with the
        exchange and K2 unless feedback=False)."""
        torch = self.torch
        self._bind(p)
        self._cur_stream = torch.cuda.current_stream(self.dev)
        st = _native.stream_ptr(self._cur_stream)
        self._control_front(st)
        self._control_back(st)
        if feedback:
            if self.world > 1:
                torch.distributed.all_reduce(self.slots, group=self.pg)
            self.step_feedback()

    def _pipe_forward(self, p):
        """Forward tail of the step in set p, on the forward stream."""
        self._bind(p)
        with self.torch.cuda.stream(self.fstream):
            self._cur_stream = self.fstream
            self._forward_tail(_native.stream_ptr(self.fstream))

    def _pipe_body(self, p):
        """Forward of the step whose control filled set p (forward stream) || the
        control of the next step into set 1 - p (current stream); joined.  Captured:
        graph(forward p) on the forward stream, graph(control 1 - p) [-> all_reduce
        -> graph(K2) for world > 1] on the serving stream."""
        torch = self.torch
        main = torch.cuda.current_stream(self.dev)
        self._fork.record(main)
        self.fstream.wait_event(self._fork)
        if self.graph is None:
            self._pipe_forward(p)
            self._pipe_control(1 - p)
        else:
            _, gf, gc, gk = self.graph
            with torch.cuda.stream(self.fstream):
                gf[p].replay()
            gc[1 - p].replay()
            if gk is not None:
                torch.distributed.all_reduce(self.slots, group=self.pg)
                gk.replay()
        self._join.record(self.fstream)
        main.wait_event(self._join)

    def flush(self) -> None:
        """Pipelined: complete the forward of the step whose control already ran."""
        if not (self.pipeline and self._ahead):
            return
        torch = self.torch
        with torch.cuda.stream(self.stream):
            self._bind(self._pset)
            self._cur_stream = self.stream
            self._forward_tail(_native.stream_ptr(self.stream))
        self._ahead = False
        self._pset ^= 1
        self.steps_run += 1
        self.stream.synchronize()

    def step_feedback(self):
        """K2 over every rank's slot (after the exchange)."""
        torch, lib, ctl = self.torch, self.lib, self.ctl
        st = _native.stream_ptr(torch.cuda.current_stream(self.dev))
        _native.check("gg_outcome_slots", lib.gg_outcome_slots(
            C.byref(ctl.params), _native.ptr(ctl.state), _native.ptr(self.slots), self.world,
            self.B, self.rank, _native.ptr(self.fifo), _native.ptr(self.err), st))

    # ------------------------------------------------------------------ graphs
    def capture(self) -> None:
        with self.torch.cuda.nvtx.range("gg.serve.capture"):
            self._capture()

    def _capture(self) -> None:
        """Capture one step as CUDA graph(s) (after one eager warm-up step).

        Single GPU: the whole step is one graph.  Multi-GPU: the local part and
        the feedback part are two graphs and the NCCL all_reduce of the
        exchange buffer runs between them on the same stream (no collective
        inside a captured graph, so any NCCL/torch combination works)."""
        torch = self.torch
        if self.pipeline:
            # per buffer set: the forward tail (forward stream) and the control chain
            # (serving stream; with K2 on one GPU, else K2 is its own graph after the
            # exchange); _pipe_body forks / joins the two streams around the replays
            gf, gc = [], []
            l0 = _native.LAUNCHES
            prev = self.lib.gg_set_sm_reserve(self.sm_reserve)
            if prev < 0:
                raise ValueError(f"invalid SM reservation {self.sm_reserve}")
            for p in (0, 1):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=self.fstream):
                    self._pipe_forward(p)
                gf.append(g)
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=self.stream):
                    self._pipe_control(p, feedback=self.world == 1)
                gc.append(g)
            self.lib.gg_set_sm_reserve(prev)
            n0 = _native.LAUNCHES
            gk = None
            if self.world > 1:
                gk = torch.cuda.CUDAGraph()
                with torch.cuda.graph(gk, stream=self.stream):
                    self.step_feedback()
            self.graph = ("pipe", tuple(gf), tuple(gc), gk)
            self.launches_per_step = (n0 - l0) // 2 + (_native.LAUNCHES - n0)
            return
        if self.world == 1:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=self.stream):
                self.step()
            self.graph = (g,)
        else:
            ga, gb = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
            with torch.cuda.graph(ga, stream=self.stream):
                self.step_local()
            with torch.cuda.graph(gb, stream=self.stream):
                self.step_feedback()
            self.graph = (ga, gb)

    def run(self, steps: int) -> None:
        with self.torch.cuda.nvtx.range(f"gg.serve.run[{steps}]"):   # host-side phase marker
            self._run(steps)

    def _run(self, steps: int) -> None:
        torch = self.torch
        if self.pipeline:
            with torch.cuda.stream(self.stream):
                for _ in range(steps):
                    if not self._ahead:   # prologue: the first step's control chain
                        self._pipe_control(self._pset)
                        self._ahead = True
                        self.control_steps += 1
                    self._pipe_body(self._pset)
                    self.control_steps += 1
                    self._pset ^= 1
            self.steps_run += steps
            return
        self.control_steps += steps
        with torch.cuda.stream(self.stream):   # replay() launches on the current stream
            for _ in range(steps):
                if self.graph is None:
                    self.step()
                elif len(self.graph) == 1:
                    self.graph[0].replay()
                else:
                    self.graph[0].replay()
                    torch.distributed.all_reduce(self.slots, group=self.pg)
                    self.graph[1].replay()
        self.steps_run += steps

    # ------------------------------------------------------------------ host views
    def record(self, step: int) -> dict:
        """The published record of device step `step` (publish=True), read from pinned
        host memory -- valid once the step has completed (e.g. after an event on
        the serving stream recorded behind it) and before step + 2 runs."""
        import numpy as np
        if not self.publish:
            raise RuntimeError("GatedServer(publish=True) writes step records")
        raw = self.host_records.numpy()[(step & 1) * self.rec_bytes:((step & 1) + 1) * self.rec_bytes]
        hdr = _abi.gg_step_record.from_buffer_copy(raw[:C.sizeof(_abi.gg_step_record)].tobytes())
        if hdr.step != step:
            raise RuntimeError(f"record slot holds step {hdr.step}, not {step}")
        B, h = self.B, C.sizeof(_abi.gg_step_record)
        co = (h + 4 * B + 7) & ~7
        n = int(hdr.count)
        return {"count": n, "window_start": int(hdr.window_start),
                "pred": raw[h:h + 4 * B].view(np.int32)[:n].copy(),
                "conf": raw[co:co + 8 * B].view(np.float64)[:n].copy(),
                "decision": raw[co + 8 * B:co + 8 * B + int(hdr.n_decided)].copy()}

    def fifo_state(self) -> _abi.gg_fifo:
        self.stream.synchronize()   # the FIFO is written by work queued on the serving stream
        return _abi.gg_fifo.from_buffer_copy(bytes(self.fifo.cpu().numpy().tobytes()))

    def done(self) -> bool:
        """Trace decided and FIFO empty (pipelined: the pending forward is then flushed)."""
        f = self.fifo_state()
        fin = f.cursor >= f.trace_len and f.tail == f.head
        if fin:
            self.flush()
        return fin

    def drain(self, max_steps: int = 1 << 30) -> int:
        """Run steps until the trace is decided and the FIFO is empty."""
        n = 0
        while not self.done() and n < max_steps:
            chunk = 8
            self.run(chunk)
            self.torch.cuda.synchronize()
            n += chunk
        return n

    def results(self) -> dict:
        f = self.fifo_state()
        st = self.ctl.state_struct()
        return {"decided": int(f.cursor), "admitted": int(f.tail), "served": int(f.head),
                "queue_depth": int(f.tail - f.head), "overflow": int(f.overflow),
                "clock": f.clock,
                "admitted_total": int(st.admitted_total), "skipped_total": int(st.skipped_total),
                "outcomes_total": int(st.outcomes_total), "ewma_joules": st.ewma_joules_per_request,
                "p95_ms": st.p95_current}


    def summary(self, label: str = "run", grid_intensity: float = 0.5) -> dict:
        """The reference's SummaryRow (telemetry.py:87-128) over the decided rows:
        skipped requests complete at arrival through the fallback (latency 0,
        zero joules); admitted ones carry their served latency; accuracy from the
        fallback accounting (needs labels/coins); makespan in trace time.  Energy
        is the modeled ledger total (EnergyLedger.total_joules)."""
        import math
        import numpy as np
        f = self.fifo_state()
        n = int(f.cursor)
        if n == 0:
            raise ValueError("empty trace")
        dec = self.decision[:n].cpu().numpy()
        lat = self.latency[:n].cpu().numpy()
        arr = self.now[:n].cpu().numpy()
        adm = (dec == _abi.GG_DECISION_DIRECT) | (dec == _abi.GG_DECISION_BATCHED)
        served = self.predicted[:n].cpu().numpy() >= 0
        lat = np.where(adm, lat, 0.0)
        finish = arr + lat / 1000.0
        mean = float(sum(lat.tolist()) / n)
        var = float(sum((x - mean) ** 2 for x in lat.tolist()) / n)
        makespan = float(finish.max() - arr.min())
        st = self.ctl.state_struct()
        joules = float(st.total_joules)
        kwh = joules / 3.6e6
        correct = int(self.correct[:n].sum().item()) if self.labels is not None else None
        return {"label": label, "avg_latency_ms": mean, "std_latency_ms": math.sqrt(var),
                "throughput_rps": n / makespan if makespan > 0 else math.inf,
                "total_time_s": makespan, "energy_kwh": kwh, "co2_kg": kwh * grid_intensity,
                "admitted_count": int(adm.sum()), "skipped_count": int(n - adm.sum()),
                "served_count": int(served.sum()),
                "accuracy": None if correct is None else correct / n}


def fallback_coins(seed: int, n: int):
    """The simulator's fallback coin stream (servesim.py:177-180, 254): the third
    child of SeedSequence(seed), one U[0, 1) draw per coin, host-side numpy."""
    import numpy as np
    rng = np.random.default_rng(np.random.SeedSequence(seed).spawn(3)[2])
    return rng.random(n)


def synthetic_images(n: int, image: int = 224, seed: int = 0, device="cuda"):
    """Resident pool of uint8 HWC images (synthetic; no dataset offline)."""
    import torch
    g = torch.Generator(device="cpu").manual_seed(seed)
    return torch.randint(0, 256, (n, image, image, 3), generator=g, dtype=torch.uint8).to(device)


def synthetic_tokens(n: int, seq_len: int = 128, vocab: int = 30522, seed: int = 0, device="cuda"):
    """Resident pool of token-id sequences + all-ones masks (synthetic)."""
    import torch
    g = torch.Generator(device="cpu").manual_seed(seed)
    ids = torch.randint(0, vocab, (n, seq_len), generator=g, dtype=torch.int32)
    return ids.to(device), torch.ones((n, seq_len), dtype=torch.int32, device=device)


def smoke():
    """Tiny closed loop on cuda:0 (ResNet-18, B=8, 64 requests, 12 decided per step).
    Returns (server, steps, scores, now) so the caller can replay the same steps
    on the host oracle (__graft_entry__.smoke; the product never imports it)."""
    import numpy as np
    import torch

    from . import controller as gcontrol
    from .energy import EnergyLedger
    from .resnet18 import ResNet18B200, random_model
    from .workload import ArrivalMode, WorkloadConfig, generate_trace

    wl = WorkloadConfig(mode=ArrivalMode.CLOSED, num_requests=64, num_classes=1000,
                        confidence_low=0.3, confidence_high=0.9)
    tr = generate_trace(wl, 1.0, np.random.default_rng(0))
    now = np.arange(64) * 0.01
    cfg = gcontrol.ControllerConfig(alpha=1.0, beta=-0.2, gamma=-0.3, tau0=0.6, tau_inf=0.3, k=2.0,
                                    routing=gcontrol.RoutePolicy.ALL_BATCHED)
    ctl = cfg.build(EnergyLedger())
    net = ResNet18B200(random_model(0), max_batch=8)
    srv = GatedServer(ctl, net, torch.from_numpy(tr.scores).cuda(), torch.from_numpy(now).cuda(),
                      synthetic_images(16), window=12)
    srv.run(1)
    srv.capture()
    steps = 1
    while not srv.done():
        srv.run(1)
        steps += 1
    torch.cuda.synchronize()
    r = srv.results()
    assert r["decided"] == 64 and r["served"] == r["admitted"] and r["overflow"] == 0, r
    pred = srv.predicted.cpu().numpy()
    dec = srv.decision.cpu().numpy()
    assert ((pred >= 0) == ((dec == 1) | (dec == 2))).all(), "served set != admitted set"
    print(f"smoke: closed loop ok ({r['admitted']}/64 admitted and served in batches of <= 8, "
          f"{steps} steps)")
    return srv, steps, tr.scores, now
