"""A few eager serving steps (for ncu launch lists): python tools/serve_once.py resnet18|distilbert [steps]"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402


def main():
    import bench
    import paper_2601_04250_b200 as gg
    from paper_2601_04250_b200 import serving

    which = sys.argv[1] if len(sys.argv) > 1 else "resnet18"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    wl = bench.WORKLOADS[which]
    scores, now = bench.make_trace(wl, (steps + 4) * wl["window"], seed=1000)
    net = bench.build_net(which, wl["batch"])
    ctl = gg.ControllerConfig(**wl["ctl"], routing=gg.RoutePolicy.ALL_BATCHED).build(gg.EnergyLedger())
    pay = serving.synthetic_images(wl["pool"]) if which == "resnet18" else serving.synthetic_tokens(wl["pool"])
    srv = serving.GatedServer(ctl, net, torch.from_numpy(scores).cuda(), torch.from_numpy(now).cuda(),
                              pay, window=wl["window"], outcome=serving.OutcomeModel(**wl["outcome"]))
    srv.run(steps)
    torch.cuda.synchronize()
    print(srv.results())


if __name__ == "__main__":
    main()
