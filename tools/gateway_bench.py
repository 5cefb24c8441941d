"""Gateway decide throughput: C concurrent clients through GatewayBatcher (coalesced
K1 launches) vs one controller.decide() per request (one K1 launch + sync each).
K = 4 scores per request.  Host-side front end on one GPU; not a bench.py number.

    python tools/gateway_bench.py [clients] [requests]
"""
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import paper_2601_04250_b200 as gg
    from paper_2601_04250_b200.gateway import GatewayBatcher
    clients = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 4000
    rng = np.random.default_rng(0)
    x = rng.random((n, 4))
    x /= x.sum(1, keepdims=True)
    bodies = [{"id": f"r{i}", "scores": x[i].tolist(), "timestamp_s": 1.0 + i * 1e-3} for i in range(n)]
    cfg = gg.ControllerConfig(alpha=1.0, beta=-0.1, gamma=-0.3, tau0=0.9, tau_inf=0.3, k=0.05)
    # sequential reference-style gateway: one decide() per request under a lock
    ctl = cfg.build(gg.EnergyLedger())
    for b in bodies[:50]:
        ctl.decide(gg.RequestFeatures(0, b["timestamp_s"], tuple(b["scores"]), None), b["timestamp_s"])
    t0 = time.perf_counter()
    for b in bodies:
        ctl.decide(gg.RequestFeatures(0, b["timestamp_s"], tuple(b["scores"]), None), b["timestamp_s"])
    seq = n / (time.perf_counter() - t0)
    with GatewayBatcher(cfg, max_wait_s=100e-6) as gw:
        for b in bodies[:200]:
            gw.decide(b)
        parts = [bodies[i::clients] for i in range(clients)]
        l0 = gw.launches["decide"]
        t0 = time.perf_counter()
        ts = [threading.Thread(target=lambda p=p: [gw.decide(b) for b in p]) for p in parts]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        bat = n / (time.perf_counter() - t0)
        launches = gw.launches["decide"] - l0
    print(f"{n} decides, K=4: sequential decide() {seq:.0f}/s; GatewayBatcher with {clients} clients "
          f"{bat:.0f}/s in {launches} K1 launches ({n / max(1, launches):.1f} requests per launch)")


if __name__ == "__main__":
    main()
