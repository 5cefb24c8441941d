"""World-size-2 test of the K9 exchange protocol on CPU (gloo).

Each process is one rank: it decides its shard with the C oracle standing in
for K1, packs its exchange slot in the device layout (GG_SLOT_LEN), all-reduces
the rank-slotted fp64 buffer with SUM over gloo (== allgather, exactly), and
applies every slot as gg_outcome_slots does.  Both replicas must end
byte-identical and equal the single-process replay of the data-parallel
semantics (oracle/serving_oracle.py).
"""

from __future__ import annotations

import os
import socket

import numpy as np
import torch.multiprocessing as mp

from tests import _golden as G

MODEL = dict(batch_base_ms=4.0, per_item_ms=0.05, batch_base_energy_j=6.0, per_item_energy_j=1.5)
PARAMS = dict(alpha=1.0, beta=-0.2, gamma=-0.4, tau0=0.8, tau_inf=0.35, k=1.5, ewma_lambda=0.9,
              direction=0, utility_proxy=0, routing=1, queue_threshold=4, p95_window=100)
B, W = 8, 14


def shards():
    out = []
    for seed in (5, 6):
        rng = np.random.default_rng(seed)
        c = rng.uniform(0.5, 1.0, size=200)
        out.append((np.stack([c, 1.0 - c], axis=1), np.arange(200) * 0.01))
    return out


def apply_slots(orc, base, slots, rank, G_):
    """Host mirror of gg_outcome_slots: other ranks' admission effects, then outcomes."""
    from oracle import serving_oracle as so
    st = orc.state
    for g in range(G_):
        if g == rank:
            continue
        sl = slots[g * (3 * B + 8) + 3 * B: (g + 1) * (3 * B + 8)]
        if sl[2] - sl[3] > 0:
            other = type(st).from_buffer_copy(bytes(base))
            # observe of this rank's snapshot (energy observe uses the replicated EWMA)
            from oracle.c_oracle import COracle
            tmp = COracle(orc.params)
            tmp.state = other
            tmp.admit(np.array([[0.5, 0.5]]), np.array([0.0]), (int(sl[6]), float(sl[7]), 0.0),
                      want_breakdown=False)
            for name in ("n_energy", "n_queue_depth", "n_p95_ms"):
                so._merge_channel(getattr(st, name), getattr(tmp.state, name))
        st.admitted_total += int(sl[4])
        st.skipped_total += int(sl[5])
    for g in range(G_):
        sl = slots[g * (3 * B + 8): (g + 1) * (3 * B + 8)]
        n = int(sl[3 * B])
        if n:
            orc.outcome(sl[:n].copy(), sl[B:B + n].copy(), sl[2 * B:2 * B + n].astype(np.int32),
                        set_queue_depth=True)


def worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    from collections import deque

    from oracle.c_oracle import COracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p = G.abi_params(PARAMS)
    orc = COracle(p)
    scores, now = shards()[rank]
    fifo, cursor, extra, steps = deque(), 0, 0, 0
    while True:
        base = type(orc.state).from_buffer_copy(bytes(orc.state))
        depth = len(fifo)
        snap = (depth + extra, orc.state.p95_current, min(1.0, depth / B))
        c1 = min(len(scores), cursor + W)
        n_dec = c1 - cursor
        info = None
        if n_dec:
            _dec, _bd, idx, info = orc.admit(scores[cursor:c1], now[cursor:c1], snap,
                                             want_breakdown=False)
            fifo.extend(cursor + int(i) for i in idx)
        cursor = c1
        n = min(B, len(fifo))
        for _ in range(n):
            fifo.popleft()
        slots = torch.zeros(world * (3 * B + 8), dtype=torch.float64)
        sl = slots[rank * (3 * B + 8):]
        dn = float(n if n else 1)
        sl[:n] = MODEL["batch_base_ms"] + MODEL["per_item_ms"] * dn
        sl[B:B + n] = (MODEL["batch_base_energy_j"] + MODEL["per_item_energy_j"] * dn) / dn
        sl[2 * B:2 * B + n] = float(len(fifo) + extra)
        sl[3 * B] = n
        sl[3 * B + 1] = len(fifo)
        if info is not None:
            sl[3 * B + 2:3 * B + 8] = torch.tensor([info.n_decided, info.n_invalid, info.n_admitted,
                                                    info.n_skipped, info.snap_queue_depth,
                                                    info.snap_p95_ms], dtype=torch.float64)
        dist.all_reduce(slots)
        arr = slots.numpy()
        apply_slots(orc, base, arr, rank, world)
        extra = int(sum(arr[g * (3 * B + 8) + 3 * B + 1] for g in range(world) if g != rank))
        steps += 1
        done = torch.tensor([1.0 if (cursor >= len(scores) and not fifo) else 0.0])
        dist.all_reduce(done)
        if done.item() == world:
            break
    q.put((rank, bytes(orc.state), steps))
    dist.destroy_process_group()


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_rank_gloo_exchange():
    from oracle import serving_oracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r, (st, n)) for r, st, n in (q.get(timeout=120) for _ in range(2)))
    for p in procs:
        p.join(timeout=60)
    (s0, n0), (s1, n1) = res[0], res[1]
    assert s0 == s1, "replicas diverged"
    _dec, _served, st = serving_oracle.replay(G.abi_params(PARAMS), shards(), W, B, MODEL, n0)
    from paper_2601_04250_b200 import _abi
    got = G.state_dict_of_abi(_abi.gg_state.from_buffer_copy(s0))
    assert got == G.state_dict_of_abi(st)
