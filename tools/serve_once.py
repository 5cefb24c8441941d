"""A few eager serving steps (for ncu launch lists): python tools/serve_once.py resnet18|distilbert [steps]"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402


def main():
    import bench

    which = sys.argv[1] if len(sys.argv) > 1 else "resnet18"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    wl = bench.WORKLOADS[which]
    dev = torch.device("cuda", 0)
    scores, now, labels = bench.make_trace(wl, (steps + 4) * wl["window"], seed=1000)
    net = bench.build_net(which, wl["batch"])
    pay = bench.payload_pool(which, wl["pool"], 0, dev)
    srv = bench.make_server(wl, which, net, torch.from_numpy(scores).to(dev), torch.from_numpy(now).to(dev),
                            torch.from_numpy(labels).to(dev), pay, dev)
    srv.run(steps)
    torch.cuda.synchronize()
    print(srv.results())


if __name__ == "__main__":
    main()
