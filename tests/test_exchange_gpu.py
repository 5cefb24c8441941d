"""Multi-rank controller exchange (K9 semantics) emulated with two ranks on one GPU.

Two GatedServers (rank 0 / rank 1 of world 2) run their local steps, their
exchange slots are summed (what NCCL all_reduce(SUM) does over NVLink), and
each applies all slots.  The replicas must stay byte-identical and equal the
host replay of the data-parallel semantics (oracle/serving_oracle.py).
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import serving_oracle
from tests import _golden as G
from tests.test_serving_gpu import MODEL, make_trace

pytestmark = pytest.mark.gpu


def test_two_rank_exchange_on_one_gpu():
    import torch
    import paper_2601_04250_b200 as gg
    from paper_2601_04250_b200 import serving
    from paper_2601_04250_b200.resnet18 import ResNet18B200, random_model

    B, W = 8, 14
    kw = dict(alpha=1.0, beta=-0.2, gamma=-0.4, tau0=0.8, tau_inf=0.35, k=1.5,
              routing=gg.RoutePolicy.ALL_BATCHED)
    net = ResNet18B200(random_model(0), max_batch=B)
    shards = [make_trace(150, 1000, seed=s) for s in (5, 6)]
    srvs = []
    for rank, (sc, nw) in enumerate(shards):
        ctl = gg.ControllerConfig(**kw).build(gg.EnergyLedger())
        srvs.append(serving.GatedServer(ctl, net, torch.from_numpy(sc).cuda(),
                                        torch.from_numpy(nw).cuda(), serving.synthetic_images(16),
                                        window=W, outcome=serving.OutcomeModel(**MODEL),
                                        fifo_capacity=1024, rank=rank, world=2))
    steps = 0
    while not all(s.done() for s in srvs) or steps == 0:
        for s in srvs:
            s.step_local()
        total = srvs[0].slots + srvs[1].slots
        for s in srvs:
            s.slots.copy_(total)
            s.step_feedback()
        torch.cuda.synchronize()
        steps += 1
        a, b = (bytes(s.ctl.state_struct()) for s in srvs)
        assert a == b, f"replicas diverged at step {steps}"
    p = G.abi_params(dict(alpha=1.0, beta=-0.2, gamma=-0.4, tau0=0.8, tau_inf=0.35, k=1.5,
                          ewma_lambda=0.9, direction=0, utility_proxy=0, routing=1,
                          queue_threshold=4, p95_window=100))
    dec_o, served_o, st_o = serving_oracle.replay(p, shards, W, B, MODEL, steps)
    for g, s in enumerate(srvs):
        assert np.array_equal(s.decision.cpu().numpy(), dec_o[g])
        pred = s.predicted.cpu().numpy()
        assert set(np.nonzero(pred >= 0)[0]) == set(served_o[g])
    assert G.state_dict_of_abi(srvs[0].ctl.state_struct()) == G.state_dict_of_abi(st_o)
