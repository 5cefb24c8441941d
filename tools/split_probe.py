"""Probe: one full-batch forward vs the batch split into halves on concurrent streams.

Every forward kernel is a persistent grid of one 227-KB CTA per SM, so at each kernel
boundary the SMs idle through the predecessor's drain and the successor's fill.  With two
independent half batches on two streams, the other stream's pending kernel can take the
SMs a draining kernel frees.  Times CUDA-graph replays with CUDA events (burst of 5 after
an idle gap, and 20 back to back), like bench.py's roofline.

    python tools/split_probe.py [resnet18|distilbert] [splits]
"""

import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402


def build(which, B):
    if which == "resnet18":
        from paper_2601_04250_b200.resnet18 import ResNet18B200, random_model
        net = ResNet18B200(random_model(0), max_batch=B)
        x = torch.randn((B, 3, 224, 224), device="cuda")
        net.forward(x)
        return net, (lambda s: net.forward_s2d(B, stream=s)), net
    from paper_2601_04250_b200.distilbert import DistilBertB200, random_model
    net = DistilBertB200(random_model(0), max_batch=B)
    ids = torch.randint(0, 30522, (B, 128), device="cuda", dtype=torch.int32)
    return net, (lambda s: net.forward(ids, stream=s)), net


def capture(fns):
    main = torch.cuda.Stream()
    side = [torch.cuda.Stream() for _ in fns]
    for _ in range(2):
        with torch.cuda.stream(main):
            for f in fns:
                f(main)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=main):
        if len(fns) == 1:
            fns[0](main)
        else:
            start = torch.cuda.Event()
            start.record(main)
            ends = []
            for f, s in zip(fns, side):
                s.wait_event(start)
                with torch.cuda.stream(s):
                    f(s)
                e = torch.cuda.Event()
                e.record(s)
                ends.append(e)
            for e in ends:
                main.wait_event(e)
    torch.cuda.synchronize()
    return g


def timeit(g, reps):
    s = torch.cuda.current_stream()
    g.replay()
    torch.cuda.synchronize()
    time.sleep(0.05)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(reps):
        g.replay()
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "resnet18"
    splits = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    B = 64 if which == "resnet18" else 128
    _, f_full, _ = build(which, B)
    parts = [build(which, B // splits) for _ in range(splits)]
    g1 = capture([f_full])
    g2 = capture([p[1] for p in parts])
    for label, g in (("full", g1), (f"{splits}x split", g2), ("full", g1), (f"{splits}x split", g2)):
        burst = sorted(timeit(g, 5) for _ in range(3))[1]
        b2b = timeit(g, 20)
        print(f"{which} B={B} {label:>9}: burst {burst * 1e3:8.1f} us   20 back-to-back {b2b * 1e3:8.1f} us",
              flush=True)


if __name__ == "__main__":
    main()
