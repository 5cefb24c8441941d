"""Run ONE hot kernel a few times at bench scale, for `ncu --set full` captures.

    python tools/kernel_probe.py k1|span1|span2|span3|span4|stem [reps]

Prints CUDA-event device times (probe numbers, not bench values).
"""

from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402


def _time(fn, reps):
    """Device time per call: the reps calls are captured in one CUDA graph and
    replayed, so host-side launch cost (ctypes, tensor-map encoding) is excluded."""
    import os
    fn()
    torch.cuda.synchronize()
    if os.environ.get("GG_SPAN_PROF") or os.environ.get("GG_PROBE_EAGER"):   # eager launches
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        return float("nan")
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def k1(reps):
    import paper_2601_04250_b200 as gg
    n = 1 << 26
    c = torch.rand(n, device="cuda", dtype=torch.float64) * 0.5 + 0.5
    scores = torch.stack([c, 1.0 - c], dim=1).contiguous()
    now = torch.linspace(0.0, 10.0, n, device="cuda", dtype=torch.float64)
    ctl = gg.ControllerConfig(alpha=1.0, beta=-0.1, gamma=-0.3, tau0=0.9, tau_inf=0.4, k=0.5,
                              routing=gg.RoutePolicy.THRESHOLD_ON_QUEUE).build(gg.EnergyLedger())
    from paper_2601_04250_b200 import _abi
    s = _abi.gg_snapshot(3, 7.5, 0.25)   # device-resident snapshot (graph-capturable)
    snap = torch.frombuffer(bytearray(bytes(s)), dtype=torch.uint8).cuda()
    out = ctl.decide_batch(scores, now, snap, breakdown=False)
    ms = _time(lambda: ctl.decide_batch(scores, now, snap, breakdown=False, out=out), reps)
    n_adm = out.n_admitted
    nbytes = n * 25 + 4 * n_adm
    print(f"k1 n={n}: {ms:.4f} ms  {nbytes / ms / 1e6:.1f} GB/s algorithmic (25 B/row + 4 B/admitted)")


SPANS = {"span1": (64, 56, 64, 64), "span2": (64, 28, 128, 128), "span3": (64, 14, 256, 256),
         "span4": (64, 7, 512, 512)}


def span(which, reps, zero=False):
    from paper_2601_04250_b200 import _native as nat
    lib = nat.load()
    n, h, c, cout = SPANS[which]
    cnt = torch.zeros(1, dtype=torch.int32, device="cuda") if zero else None
    xp = torch.zeros((n, h + 2, h + 2, c), dtype=torch.bfloat16, device="cuda")
    xp[:, 1:-1, 1:-1] = torch.randn((n, h, h, c), device="cuda").to(torch.bfloat16)
    wk = (torch.randn((cout, 9 * c), device="cuda") / (9 * c) ** 0.5).to(torch.bfloat16)
    b = torch.zeros(cout, device="cuda")
    y = torch.zeros((n, h + 2, h + 2, cout), dtype=torch.bfloat16, device="cuda")

    def run():
        nat.check("gg_conv3x3_padded", lib.gg_conv3x3_padded(
            nat.ptr(xp), n, h, h, c, nat.ptr(wk), cout, nat.ptr(b), None, 1, nat.ptr(y),
            nat.ptr(cnt), nat.stream_ptr()))
    ms = _time(run, reps)
    fl = 2.0 * n * h * h * cout * 9 * c
    print(f"{which} {n}x{h}x{h}x{c}->{cout}: {ms * 1e3:.1f} us  {fl / ms / 1e9:.1f} TFLOP/s")


def stem(reps):
    from paper_2601_04250_b200 import _native as nat
    lib = nat.load()
    n = 64
    x = torch.zeros((n, 115, 115, 16), dtype=torch.bfloat16, device="cuda")
    x[:, 2:-1, 2:-1, :12] = torch.randn((n, 112, 112, 12), device="cuda").to(torch.bfloat16)
    w = (torch.randn((64, 256), device="cuda") / 16).to(torch.bfloat16)
    b = torch.zeros(64, device="cuda")
    y = torch.empty((n, 112, 112, 64), dtype=torch.bfloat16, device="cuda")

    def run():
        nat.check("gg_stem_s2d_span", lib.gg_stem_s2d_span(
            nat.ptr(x), n, 112, 112, nat.ptr(w), 64, nat.ptr(b), 1, nat.ptr(y), None,
            nat.stream_ptr()))
    ms = _time(run, reps)
    fl = 2.0 * n * 112 * 112 * 64 * 147
    print(f"stem span {n}x112x112: {ms * 1e3:.1f} us  {fl / ms / 1e9:.1f} TFLOP/s (7x7x3 algorithmic)")


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "k1"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    if which == "k1":
        k1(reps)
    elif which in SPANS:
        span(which, reps)
    elif which.endswith("z") and which[:-1] in SPANS:   # count = 0: fixed launch cost
        span(which[:-1], reps, zero=True)
    elif which == "stem":
        stem(reps)
    else:
        raise SystemExit(f"unknown probe {which}")


if __name__ == "__main__":
    main()
