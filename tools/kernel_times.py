"""Per-kernel device times of one warm forward, in launch order, via torch.profiler (CUPTI
activity records; kernels run back to back as in the real step, not serialised like ncu).

    python tools/kernel_times.py resnet18|distilbert [reps]

Not a bench number: a breakdown to decide what to optimise next."""

import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "resnet18"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    if which == "resnet18":
        from paper_2601_04250_b200.resnet18 import ResNet18B200, random_model
        net = ResNet18B200(random_model(0), max_batch=64)
        x = torch.randn((64, 3, 224, 224), device="cuda")
        fwd = lambda: net.forward(x)  # noqa: E731
        flops = net.flops(64)
    else:
        from paper_2601_04250_b200.distilbert import DistilBertB200, random_model
        net = DistilBertB200(random_model(0), max_batch=128)
        ids = torch.randint(0, 30522, (128, 128), device="cuda", dtype=torch.int32)
        fwd = lambda: net.forward(ids)  # noqa: E731
        flops = net.flops(128)
    for _ in range(5):
        fwd()
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(reps):
            fwd()
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    evs.sort(key=lambda e: e.time_range.start)
    per = len(evs) // reps
    last = evs[-per:]
    t0 = last[0].time_range.start
    span = last[-1].time_range.end - t0
    print(f"{which}: {per} kernels/forward; last forward span {span:.1f} us "
          f"({flops / span / 1e6:.1f} TFLOP/s algorithmic)")
    busy = 0.0
    for e in last:
        d = e.time_range.end - e.time_range.start
        busy += d
        print(f"  {e.time_range.start - t0:8.1f} {d:8.2f}  {e.name[:110]}")
    print(f"  sum of kernel durations {busy:.1f} us (gaps {span - busy:.1f} us)")
    agg = defaultdict(lambda: [0, 0.0])
    for e in evs:
        a = agg[e.name[:90]]
        a[0] += 1
        a[1] += e.time_range.end - e.time_range.start
    print("aggregate (all reps):")
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"  {t / reps:9.1f} us/fwd  {n // reps:3d}x  {k}")


if __name__ == "__main__":
    main()
