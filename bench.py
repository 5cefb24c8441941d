#!/usr/bin/env python
"""Benchmark of the gated-inference hot path (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload resnet18|distilbert]

Metric (BASELINE.json): admitted inferences/sec — requests that passed the
admission controller AND completed a forward pass, per second, whole job.

One step = one closed-loop serving step (serving.GatedServer): K1 admission
of `window` new arrivals against the device FIFO's congestion snapshot, pop
up to B admitted requests, gather their payloads, forward (ResNet-18 224x224,
B = 64 | DistilBERT seq 128, B = 128), K3 epilogue, outcome record, (K9
exchange for N > 1), K2 feedback.  Captured once as a CUDA graph and replayed.

  value   device-resident trace + payload pool, graph replays, CUDA events,
          max over ranks.
  e2e     same loop through the public API with host buffers: every step
          copies the window's scores/now and payload images from pinned host
          memory and reads back the served batch's predictions.
  roofline  the forward pass (the dominant kernel family: ~90 % of a step),
          algorithmic FLOPs / CUDA-event time of a full batch, vs the measured
          sustained bf16 peak (MEASURED_PEAKS.json); traffic = the DRAM bytes of
          one full-batch forward from the committed ncu launch list
          (profiles/r1g_forward_traffic.json).
  cpu_baseline / --impl reference
          the reference's CPU path: the controller port (oracle/, the
          reference's algorithm in CPython) deciding the same windows, plus a
          torch-eager fp32 CPU forward of the admitted requests as the stand-in
          for the inference the reference only simulates, on all host cores.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # BASELINE.json configs[1]: ResNet-18 224x224 gated inference, batch 64
    "resnet18": dict(batch=64, window=112, k=1000, conf_lo=0.3, conf_hi=0.9, pool=2048,
                     ctl=dict(alpha=1.0, beta=-0.1, gamma=-0.3, tau0=0.35, tau_inf=0.35, k=1.0),
                     outcome=dict(batch_base_ms=4.0, per_item_ms=0.05, batch_base_energy_j=6.0,
                                  per_item_energy_j=1.5)),
    # BASELINE.json configs[2]: DistilBERT seq 128 gated inference, batch 128, bf16
    "distilbert": dict(batch=128, window=224, k=2, conf_lo=0.85, conf_hi=0.97, pool=4096,
                       ctl=dict(alpha=1.0, beta=-0.1, gamma=-0.3, tau0=0.39796077431433013,
                                tau_inf=0.39796077431433013, k=1.0),
                       outcome=dict(batch_base_ms=4.0, per_item_ms=0.02, batch_base_energy_j=6.0,
                                    per_item_energy_j=1.0)),
}


def peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return {"hbm": d["hbm_gbs"], "bf16": d["bf16_tflops"],
                "bf16_sustained": d.get("bf16_tflops_sustained", d["bf16_tflops"]),
                "source": "measured"}
    except Exception:
        return {"hbm": 6650.0, "bf16": 1590.0, "bf16_sustained": 1400.0, "source": "fallback"}


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = str(gpu_index)
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, power, reasons = [], None, [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9 or parts[0] != self.idx:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
                power.append(float(parts[3]))
            except ValueError:
                continue
            for name, val in zip(names, parts[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": smax, "reasons": ["no samples"]}
        load = [s for s, p in zip(sm, power) if p > 0.5 * max(power)] or sm
        return {"sm_mhz": statistics.median(load), "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- setup
def make_trace(wl: dict, n: int, seed: int):
    import numpy as np
    import paper_2601_04250_b200 as gg
    cfg = gg.WorkloadConfig(mode=gg.ArrivalMode.POISSON, rate_rps=20000.0, num_classes=wl["k"],
                            confidence_low=wl["conf_lo"], confidence_high=wl["conf_hi"])
    horizon = 1.5 * n / 20000.0 + 1.0
    tr = gg.generate_trace(cfg, horizon, np.random.default_rng(seed))
    assert len(tr) >= n, (len(tr), n)
    return tr.scores[:n].copy(), tr.arrival_t[:n].copy()


def build_net(name: str, B: int):
    if name == "resnet18":
        from paper_2601_04250_b200.resnet18 import ResNet18B200, random_model
        return ResNet18B200(random_model(0), max_batch=B)
    from paper_2601_04250_b200.distilbert import DistilBertB200, random_model
    return DistilBertB200(random_model(0), max_batch=B)


# ----------------------------------------------------------------------------- our arm
def run_ours(args, wl, rank, world, local_rank, pg):
    import numpy as np
    import torch
    import paper_2601_04250_b200 as gg
    from paper_2601_04250_b200 import _native, serving

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    B, W = wl["batch"], wl["window"]
    e2e_steps = args.steps
    n_rows = (args.warmup + 2 + args.steps + args.warmup + e2e_steps + 4) * W
    scores_np, now_np = make_trace(wl, n_rows, seed=1000 + rank)
    net = build_net(args.workload, B)
    ctl = gg.ControllerConfig(**wl["ctl"], routing=gg.RoutePolicy.ALL_BATCHED).build(
        gg.EnergyLedger(), device=dev)
    if args.workload == "resnet18":
        payloads = serving.synthetic_images(wl["pool"], seed=rank, device=dev)
    else:
        payloads = serving.synthetic_tokens(wl["pool"], seed=rank, device=dev)
    scores = torch.from_numpy(scores_np).to(dev)
    now = torch.from_numpy(now_np).to(dev)
    srv = serving.GatedServer(ctl, net, scores, now, payloads, window=W,
                              outcome=serving.OutcomeModel(**wl["outcome"]), rank=rank,
                              world=world, process_group=pg)
    # warm-up: one eager step (allocations, tensor-map encodes), capture, W graph steps
    srv.run(1)
    torch.cuda.synchronize()
    _native.LAUNCHES = 0
    srv.capture()
    launches_per_step = _native.LAUNCHES
    srv.run(args.warmup)
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    f0 = srv.fifo_state()
    clocks = ClockSampler(local_rank)
    clocks.start()
    barrier()
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record(srv.stream)
    srv.run(args.steps)
    end.record(srv.stream)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    ms = start.elapsed_time(end)
    f1 = srv.fifo_state()
    served = f1.head - f0.head
    decided = f1.cursor - f0.cursor
    admitted = f1.tail - f0.tail

    # ---- e2e through the public API with host buffers -----------------------
    e2e = run_e2e(srv, scores_np, now_np, payloads, wl, e2e_steps, args.warmup)

    # ---- roofline of the forward (full batch, CUDA events on the launch stream)
    ro = roofline_forward(srv, net, B)
    energy = forward_energy(srv, net, B, local_rank)
    k1 = admission_kernel_roofline(dev) if rank == 0 else None

    tot = torch.tensor([ms, float(served), float(decided), float(admitted), e2e["ms"],
                        float(e2e["served"])], dtype=torch.float64, device=dev)
    if world > 1:
        mx = tot.clone()
        torch.distributed.all_reduce(mx, op=torch.distributed.ReduceOp.MAX)
        torch.distributed.all_reduce(tot)
        ms_max, e2e_ms_max = mx[0].item(), mx[4].item()
    else:
        ms_max, e2e_ms_max = ms, e2e["ms"]
    served_all, decided_all, admitted_all = tot[1].item(), tot[2].item(), tot[3].item()
    e2e_served_all = tot[5].item()
    res = srv.results()
    return dict(ms=ms_max, served=served_all, decided=decided_all, admitted=admitted_all,
                e2e_ms=e2e_ms_max, e2e_served=e2e_served_all, e2e=e2e, roofline=ro, clocks=clk, k1=k1,
                energy=energy,
                launches_per_step=launches_per_step, overflow=res["overflow"],
                queue_depth=res["queue_depth"])


def run_e2e(srv, scores_np, now_np, payloads, wl, steps, warmup):
    """Public-API loop with host buffers, pipelined like a serving front end: the
    window of step i+1 (scores, arrival times, payload images: pinned host ->
    device on a copy stream) uploads while step i computes; every step's served
    predictions/confidences and the window's decisions come back device -> host
    and the host waits for them one step behind.  All copies are inside the
    timed region (CUDA events)."""
    import torch
    W, T = srv.W, srv.T
    f = srv.fifo_state()
    cursor = int(f.cursor)
    P = int(payloads.shape[0] if srv.kind == "resnet18" else payloads[0].shape[0])
    if srv.kind == "resnet18":
        host_pay = torch.randint(0, 256, tuple(payloads.shape[1:]), dtype=torch.uint8)
        host_pay = host_pay.unsqueeze(0).repeat(W, 1, 1, 1).pin_memory()
        dev_pay = payloads
        pay_row = host_pay[0].numel()
    else:
        host_pay = payloads[0][:W].cpu().pin_memory()
        dev_pay = payloads[0]
        pay_row = host_pay[0].numel() * 4
    host_scores = torch.from_numpy(scores_np).pin_memory()
    host_now = torch.from_numpy(now_np).pin_memory()
    outs = [dict(count=torch.empty(1, dtype=torch.int32).pin_memory(),
                 pred=torch.empty(srv.B, dtype=torch.int32).pin_memory(),
                 conf=torch.empty(srv.B, dtype=torch.float64).pin_memory(),
                 dec=torch.empty(W, dtype=torch.uint8).pin_memory()) for _ in range(2)]
    s = srv.stream
    cs = torch.cuda.Stream(device=srv.dev)
    ev_in = [torch.cuda.Event(), torch.cuda.Event()]
    ev_out = [torch.cuda.Event(), torch.cuda.Event()]
    stats = {"h2d": 0, "d2h": 0}

    def upload(c, slot):
        c1 = min(T, c + W)
        n = c1 - c
        with torch.cuda.stream(cs):
            srv.scores[c:c1].copy_(host_scores[c:c1], non_blocking=True)
            srv.now[c:c1].copy_(host_now[c:c1], non_blocking=True)
            lo, hi = c % P, c % P + n        # payloads go to their pool slots (row % P)
            if hi <= P:
                dev_pay[lo:hi].copy_(host_pay[:n], non_blocking=True)
            else:
                dev_pay[lo:].copy_(host_pay[:P - lo], non_blocking=True)
                dev_pay[: hi - P].copy_(host_pay[P - lo:n], non_blocking=True)
            ev_in[slot].record(cs)
        stats["h2d"] += n * (srv.K + 1) * 8 + n * pay_row
        return c1

    def run(nsteps, c):
        nxt = upload(c, 0)
        for i in range(nsteps):
            slot = i & 1
            s.wait_event(ev_in[slot])
            srv.run(1)
            o = outs[slot]
            n = nxt - c
            with torch.cuda.stream(s):
                o["count"].copy_(srv.count, non_blocking=True)
                o["pred"].copy_(srv.batch_pred, non_blocking=True)
                o["conf"].copy_(srv.batch_conf, non_blocking=True)
                o["dec"][:n].copy_(srv.decision[c:nxt], non_blocking=True)
                ev_out[slot].record(s)
            stats["d2h"] += 4 + srv.B * 12 + n
            c = nxt
            if i + 1 < nsteps:
                nxt = upload(c, slot ^ 1)
            if i >= 1:
                ev_out[slot ^ 1].synchronize()   # host consumes step i-1's results
        ev_out[(nsteps - 1) & 1].synchronize()
        return c

    cursor = run(warmup, cursor)
    f0 = srv.fifo_state()
    stats["h2d"] = stats["d2h"] = 0
    torch.cuda.synchronize()
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st.record(s)
    cs.wait_stream(s)
    cursor = run(steps, cursor)
    en.record(s)
    torch.cuda.synchronize()
    f1 = srv.fifo_state()
    return {"ms": st.elapsed_time(en), "served": int(f1.head - f0.head),
            "h2d_bytes_per_step": stats["h2d"] // max(1, steps),
            "d2h_bytes_per_step": stats["d2h"] // max(1, steps)}


def admission_kernel_roofline(dev, n_rows: int = 1 << 26, k: int = 2, reps: int = 10):
    """K1 alone at scale (the north star's HBM evidence): decide_batch over n_rows
    device-resident K=2 fp64 score rows with one frozen snapshot, writing the
    decision codes and the dense admitted-index list.  Algorithmic bytes per
    launch = n*(8k + 8 + 1) + 4*n_admitted; inputs (1.6 GB) exceed L2."""
    import torch
    import paper_2601_04250_b200 as gg
    g = torch.Generator(device=dev).manual_seed(7)
    c = torch.rand(n_rows, generator=g, device=dev, dtype=torch.float64) * 0.5 + 0.5
    scores = torch.stack([c, 1.0 - c], dim=1).contiguous()
    now = torch.linspace(0.0, 10.0, n_rows, device=dev, dtype=torch.float64)
    del c
    ctl = gg.ControllerConfig(alpha=1.0, beta=-0.1, gamma=-0.3, tau0=0.9, tau_inf=0.4, k=0.5,
                              routing=gg.RoutePolicy.THRESHOLD_ON_QUEUE).build(gg.EnergyLedger(),
                                                                               device=dev)
    snap = gg.CongestionSnapshot(3, 7.5, 0.25)
    out = ctl.decide_batch(scores, now, snap, breakdown=False)
    torch.cuda.synchronize()
    n_adm = out.n_admitted
    s = torch.cuda.current_stream(dev)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(reps):
        ctl.decide_batch(scores, now, snap, breakdown=False, out=out)
    b.record(s)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    nbytes = n_rows * (8 * k + 8 + 1) + 4 * n_adm
    gbs = nbytes / (ms * 1e-3) / 1e9
    pk = peaks()
    res = {"kernel": "admit_small_kernel<2> (K1: validate + entropy + J/tau + ballot compaction)",
           "rows": n_rows, "k": k, "ms_per_launch": round(ms, 4),
           "decisions_per_s": round(n_rows / (ms * 1e-3), 1), "bound": "hbm",
           "achieved": round(gbs, 1), "peak": pk["hbm"], "unit": "GB/s",
           "frac": round(gbs / pk["hbm"], 4), "bytes_per_launch": nbytes, "admitted": n_adm}
    del scores, now, out
    torch.cuda.empty_cache()
    return res


def roofline_forward(srv, net, B):
    import torch
    torch.cuda.synchronize()
    full = torch.full((1,), B, dtype=torch.int32, device=srv.dev)
    s = srv.stream
    reps = 20

    def fwd():
        if srv.kind == "resnet18":
            net.forward_s2d(B, stream=s, count=full)
        else:
            net.forward(srv.tok_ids, srv.tok_mask, batch=B, stream=s, count=full)
    with torch.cuda.stream(s):
        for _ in range(3):
            fwd()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    with torch.cuda.stream(s):
        for _ in range(reps):
            fwd()
    b.record(s)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    flops = net.flops(B)
    pk = peaks()
    achieved = flops / (ms * 1e-3) / 1e12
    kern = ("ResNet-18 forward: fused stem conv + max pool + 4 span convs (layer 1) + 9 CTA-pair "
            "span convs (layers 2-4) + 3 fused stride-2 conv/downsample (TMA im2col) + avg pool + "
            "fc, all tcgen05, shared-border NHWC layout"
            if srv.kind == "resnet18"
            else "DistilBERT forward: 24 CTA-pair tcgen05 GEMMs + 2 single-CTA GEMMs + 6 tcgen05 "
                 "attention + 12 LayerNorm + embedding-LN")
    traffic, traffic_src = None, None
    try:   # committed ncu evidence: DRAM bytes of one full-batch forward (tools/profile_round.sh)
        with open(os.path.join(ROOT, "profiles", "r1g_forward_traffic.json")) as f:
            t = json.load(f)[srv.kind]
        traffic, traffic_src = int(t["dram_bytes_per_forward"]), t["source"]
    except Exception:
        pass
    return {"bound": "tensor", "achieved": round(achieved, 2), "peak": pk["bf16_sustained"],
            "unit": "TFLOP/s", "frac": round(achieved / pk["bf16_sustained"], 4),
            "traffic": traffic, "traffic_unit": "bytes per forward (DRAM read + write)",
            "traffic_source": traffic_src, "kernel": kern, "flops_per_launch": flops,
            "ms_per_launch": round(ms, 4), "peak_source": pk["source"] + " bf16_tflops_sustained"}


def forward_energy(srv, net, B, local_rank, seconds: float = 0.5):
    """Measured energy (NVML total-energy counter, this GPU) of full-batch forwards
    replayed back to back for >= `seconds` — joules per inference of the dominant
    kernel family (telemetry).  None without NVML."""
    import time
    import torch
    from paper_2601_04250_b200.nvml_energy import NvmlEnergyMeter, NvmlUnavailable, energy_report
    try:
        meter = NvmlEnergyMeter.for_cuda_device(torch.cuda.current_device())
    except NvmlUnavailable:
        return None
    full = torch.full((1,), B, dtype=torch.int32, device=srv.dev)
    s = srv.stream
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        if srv.kind == "resnet18":
            net.forward_s2d(B, stream=s, count=full)
        else:
            net.forward(srv.tok_ids, srv.tok_mask, batch=B, stream=s, count=full)
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        for _ in range(10):
            if srv.kind == "resnet18":
                net.forward_s2d(B, stream=s, count=full)
            else:
                net.forward(srv.tok_ids, srv.tok_mask, batch=B, stream=s, count=full)
    n = 0
    torch.cuda.synchronize()
    meter.start()
    t0 = time.perf_counter()
    with torch.cuda.stream(s):
        while time.perf_counter() - t0 < seconds:
            for _ in range(20):
                g.replay()
            n += 200
            torch.cuda.synchronize()
    joules = meter.stop()
    secs = time.perf_counter() - t0
    r = energy_report(joules, float(n * B))
    r.update({"seconds": round(secs, 3), "mean_watts": round(joules / secs, 1) if secs > 0 else None,
              "scope": f"{n} full-batch forwards (B={B}) replayed back to back, NVML "
                       "nvmlDeviceGetTotalEnergyConsumption delta on this GPU; telemetry, not "
                       "fed to the controller"})
    for k in ("joules", "joules_per_inference", "kwh_per_million", "kg_co2_per_million"):
        r[k] = round(r[k], 6) if r[k] == r[k] else None
    return r


# ----------------------------------------------------------------------------- reference arm
def cpu_reference(wl: dict, workload: str, steps: int, warmup: int, sample_steps: int | None = None):
    """Reference CPU path: the controller port in CPython (oracle/controller_oracle.py,
    the reference's algorithm) deciding each window + a torch-eager fp32 CPU forward
    of the admitted requests (stand-in: the reference only simulates inference)."""
    import numpy as np
    import torch
    from oracle import controller_oracle as O

    threads = os.cpu_count() or 1
    torch.set_num_threads(threads)
    B, W = wl["batch"], wl["window"]
    n_steps = warmup + steps
    scores, now = make_trace(wl, (n_steps + 2) * W, seed=1000)
    if workload == "resnet18":
        from paper_2601_04250_b200.resnet18 import random_model
        model = random_model(0).eval()
        x_pool = torch.randn((8, 3, 224, 224))
    else:
        from paper_2601_04250_b200.distilbert import random_model
        model = random_model(0).eval()
        x_pool = torch.randint(0, 30522, (8, 128))
    c = wl["ctl"]
    ctl = O.OracleController(O.OracleParams(alpha=c["alpha"], beta=c["beta"], gamma=c["gamma"],
                                            tau0=c["tau0"], tau_inf=c["tau_inf"], k=c["k"],
                                            routing=O.ALL_BATCHED))
    fifo: list[int] = []
    m = wl["outcome"]
    served = 0
    t_total = 0.0
    for s in range(n_steps):
        t0 = time.perf_counter()
        depth = len(fifo)
        snap = (depth, ctl.p95_ms(), min(1.0, depth / B))
        rows = scores[s * W:(s + 1) * W]
        for i in range(rows.shape[0]):
            d = ctl.decide([float(v) for v in rows[i]], float(now[s * W + i]), snap)
            if d.admit:
                fifo.append(s * W + i)
        batch, fifo = fifo[:B], fifo[B:]
        n = len(batch)
        if n:
            with torch.no_grad():
                xb = x_pool[torch.arange(n) % x_pool.shape[0]]
                model(xb) if workload == "resnet18" else model(input_ids=xb)
            lat = m["batch_base_ms"] + m["per_item_ms"] * n
            jo = (m["batch_base_energy_j"] + m["per_item_energy_j"] * n) / n
            for _ in range(n):
                ctl.record_outcome(lat, jo, len(fifo))
        dt = time.perf_counter() - t0
        if s >= warmup:
            t_total += dt
            served += n
    return {"value": served / t_total, "served": served, "seconds": t_total, "cores": threads,
            "steps": steps}


# ----------------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=list(WORKLOADS), default="resnet18")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    wl = WORKLOADS[args.workload]
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    metric = "admitted inferences/sec"
    config = {"workload": f"{args.workload} gated inference, forward batch {wl['batch']}, "
                          f"{wl['window']} arrivals/step, K={wl['k']} gating scores",
              "model": args.workload, "global_batch": wl["batch"] * world,
              "seq_len": 128 if args.workload == "distilbert" else None,
              "image": 224 if args.workload == "resnet18" else None,
              "window": wl["window"], "controller": wl["ctl"],
              "parallelism": f"dp{world}" if world > 1 else "single",
              "l2": "activation working set > 126 MB L2 (no flush needed)"}

    if args.impl == "reference":
        if rank != 0:
            return
        steps = min(args.steps, 10)
        r = cpu_reference(wl, args.workload, steps, min(args.warmup, 3))
        line = {"impl": "reference", "metric": metric, "value": round(r["value"], 3),
                "unit": "inferences/s", "n_gpus": args.gpus, "steps": steps,
                "warmup": min(args.warmup, 3), "ms_per_step": round(1e3 * r["seconds"] / steps, 3),
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "fp64 controller / fp32 forward", "data": "synthetic", "config": config,
                "cpu_baseline": {"value": round(r["value"], 3), "unit": "inferences/s",
                                 "cores": r["cores"], "kind": "port",
                                 "sample": f"{steps} steps x {wl['window']} arrivals: CPython "
                                           "controller port + torch-eager fp32 CPU forward "
                                           "(stand-in; the reference simulates inference)"},
                "e2e": {"value": round(r["value"], 3), "unit": "inferences/s",
                        "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    pg = None
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        pg = dist.group.WORLD
    r = run_ours(args, wl, rank, world, local_rank, pg)
    if rank != 0:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return
    value = r["served"] / (r["ms"] * 1e-3)
    e2e_value = r["e2e_served"] / (r["e2e_ms"] * 1e-3) if r["e2e_ms"] > 0 else None
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        c = cpu_reference(wl, args.workload, steps=2, warmup=1)
        cpu = {"value": round(c["value"], 3), "unit": "inferences/s", "cores": c["cores"],
               "kind": "port",
               "sample": f"2 steps x {wl['window']} arrivals: CPython controller port + "
                         "torch-eager fp32 CPU forward (stand-in)"}
    line = {"metric": metric, "value": round(value, 2), "unit": "inferences/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(r["ms"] / args.steps, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (reference-order numpy traces, random-init weights)",
            "config": config,
            "admission_rate": round(r["admitted"] / max(1, r["decided"]), 4),
            "mean_forward_batch": round(r["served"] / (args.steps * world), 2),
            "queue_depth_end": r["queue_depth"], "fifo_overflow": r["overflow"],
            "roofline": r["roofline"], "admission_roofline": r["k1"], "cpu_baseline": cpu,
            "e2e": {"value": round(e2e_value, 2) if e2e_value else None, "unit": "inferences/s",
                    "h2d_bytes_per_step": r["e2e"]["h2d_bytes_per_step"],
                    "d2h_bytes_per_step": r["e2e"]["d2h_bytes_per_step"]},
            "gpu_launches": r["launches_per_step"] * args.steps,
            "clocks": r["clocks"],
            "energy": r["energy"]}
    print(json.dumps(line))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
