"""Two real processes, two controller replicas, the real K1/K2 kernels and a
real torch.distributed exchange.

Each process is one rank with its own GatedServer (world = 2): the serving
step is captured as the two CUDA graphs GatedServer.capture() builds for
world > 1, with the K9 all_reduce(SUM) of the rank-slotted fp64 exchange
buffer between them, exactly as bench.py --gpus N runs it.

* gloo backend, both ranks on cuda:0: runs on the single-GPU box (gloo
  all-reduces CUDA tensors through the host), so the multi-process path with
  the device kernels is exercised on every GPU test run.
* nccl backend, one GPU per rank: skipped unless >= 2 GPUs are visible.

pipe=True: the software-pipelined serving loop (GatedServer(pipeline=True):
graph(forward) on a second stream || graph(control) -> all_reduce -> graph(K2)).

Checks: the two replicas' controller states are byte-identical after every
step, and equal the host replay of the data-parallel semantics
(oracle/serving_oracle.py) together with every rank's decisions and served set.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

MODEL = dict(batch_base_ms=4.0, per_item_ms=0.05, batch_base_energy_j=6.0, per_item_energy_j=1.5)
PARAMS = dict(alpha=1.0, beta=-0.2, gamma=-0.4, tau0=0.8, tau_inf=0.35, k=1.5, ewma_lambda=0.9,
              direction=0, utility_proxy=0, routing=1, queue_threshold=4, p95_window=100)
B, W, N = 16, 40, 400


def _shard(rank):
    import paper_2601_04250_b200 as gg
    wl = gg.WorkloadConfig(mode=gg.ArrivalMode.POISSON, rate_rps=5000.0, num_classes=2,
                           confidence_low=0.55, confidence_high=0.97)
    tr = gg.generate_trace(wl, 1.0, np.random.default_rng(50 + rank))
    return tr.scores[:N].copy(), tr.arrival_t[:N].copy()


def _worker(rank, world, port, backend, q, pipe=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    import torch
    import torch.distributed as dist
    import paper_2601_04250_b200 as gg
    from paper_2601_04250_b200 import serving
    from paper_2601_04250_b200.distilbert import DistilBertB200, random_model
    try:
        dev = torch.device("cuda", rank if backend == "nccl" else 0)
        torch.cuda.set_device(dev)
        if backend == "nccl":
            dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
        else:
            dist.init_process_group("gloo", rank=rank, world_size=world)
        kw = {k: PARAMS[k] for k in ("alpha", "beta", "gamma", "tau0", "tau_inf", "k")}
        ctl = gg.ControllerConfig(**kw, routing=gg.RoutePolicy.ALL_BATCHED).build(
            gg.EnergyLedger(), device=dev)
        sc, nw = _shard(rank)
        net = DistilBertB200(random_model(0), max_batch=B, device=dev)
        srv = serving.GatedServer(ctl, net, torch.from_numpy(sc).to(dev), torch.from_numpy(nw).to(dev),
                                  serving.synthetic_tokens(32, device=dev), window=W,
                                  outcome=serving.OutcomeModel(**MODEL), fifo_capacity=1024,
                                  rank=rank, world=world, process_group=dist.group.WORLD,
                                  pipeline=pipe)
        srv.run(1)                 # eager step (exchange through the process group)
        srv.capture()              # graph(local) -> all_reduce -> graph(feedback)
        steps, diverged = 1, -1
        while True:
            torch.cuda.synchronize()
            done = torch.tensor([1.0 if srv.done() else 0.0], device=dev)
            dist.all_reduce(done)
            if done.item() == world:
                break
            srv.run(1)
            steps += 1
            torch.cuda.synchronize()
            st = srv.ctl.state.clone()
            other = [torch.empty_like(st) for _ in range(world)]
            dist.all_gather(other, st)
            if diverged < 0 and not all(torch.equal(other[0], o) for o in other):
                diverged = steps
        q.put((rank, srv.control_steps, diverged, srv.decision.cpu().numpy(),
               np.nonzero(srv.predicted.cpu().numpy() >= 0)[0], bytes(srv.ctl.state_struct()), None))
        dist.destroy_process_group()
    except Exception as exc:  # pragma: no cover - reported by the parent
        import traceback
        q.put((rank, 0, 0, None, None, None, traceback.format_exc()))
        raise


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(backend, pipe=False):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, backend, q, pipe)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
    res.sort(key=lambda r: r[0])
    for r in res:
        assert r[6] is None, r[6]
    return res


@pytest.mark.parametrize("backend,pipe", [("gloo", False), ("gloo", True), ("nccl", False),
                                          ("nccl", True)])
def test_two_process_exchange(backend, pipe):
    import torch
    from oracle import serving_oracle
    from paper_2601_04250_b200 import _abi
    from tests import _golden as G
    if backend == "nccl" and torch.cuda.device_count() < 2:
        pytest.skip("NCCL exchange needs >= 2 GPUs (one rank per GPU)")
    res = _run(backend, pipe)
    steps = res[0][1]
    assert res[1][1] == steps
    assert res[0][2] < 0 and res[1][2] < 0, "replicas diverged"
    assert res[0][5] == res[1][5]                       # byte-identical replicas
    p = G.abi_params(PARAMS)
    dec_o, served_o, st_o = serving_oracle.replay(p, [_shard(0), _shard(1)], W, B, MODEL, steps)
    for g in range(2):
        assert np.array_equal(res[g][3], dec_o[g])
        assert set(res[g][4].tolist()) == set(served_o[g])
    st = _abi.gg_state.from_buffer_copy(res[0][5])
    assert G.state_dict_of_abi(st) == G.state_dict_of_abi(st_o)
