"""Per-kernel device times of graph-replayed serving steps (CUPTI via torch.profiler),
in launch order for the last step plus an aggregate — the bench's step, broken down.

    python tools/step_times.py resnet18|distilbert [steps]

Not a bench number."""

import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402


def main():
    import bench
    import paper_2601_04250_b200 as gg
    from paper_2601_04250_b200 import serving

    which = sys.argv[1] if len(sys.argv) > 1 else "resnet18"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    wl = bench.WORKLOADS[which]
    dev = torch.device("cuda", 0)
    scores, now, labels = bench.make_trace(wl, (steps + 16) * wl["window"], seed=1000)
    net = bench.build_net(which, wl["batch"])
    pay = bench.payload_pool(which, wl["pool"], 0, dev)
    srv = bench.make_server(wl, which, net, torch.from_numpy(scores).to(dev), torch.from_numpy(now).to(dev),
                            torch.from_numpy(labels).to(dev), pay, dev)
    srv.run(1)
    srv.capture()
    srv.run(4)
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        srv.run(steps)
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    evs.sort(key=lambda e: e.time_range.start)
    per = len(evs) // steps
    last = evs[-per:]
    t0 = last[0].time_range.start
    span = last[-1].time_range.end - t0
    print(f"{which}: {per} kernels/step; last step span {span:.1f} us")
    prev_end = t0
    for e in last:
        d = e.time_range.end - e.time_range.start
        print(f"  {e.time_range.start - t0:8.1f} {d:8.2f} (+{e.time_range.end - prev_end:7.2f})  {e.name[:90]}")
        prev_end = max(prev_end, e.time_range.end)
    agg = defaultdict(lambda: [0, 0.0])
    for e in evs:
        a = agg[e.name[:80]]
        a[0] += 1
        a[1] += e.time_range.end - e.time_range.start
    print("aggregate (all steps):")
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:12]:
        print(f"  {t / steps:9.1f} us/step  {n // steps:3d}x  {k}")


if __name__ == "__main__":
    main()
