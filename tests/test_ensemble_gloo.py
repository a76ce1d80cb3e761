"""World-size-2 gloo tests (CPU) of the ensemble sharding host logic."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

from paper_1611_06721_b200 import ensemble as E


def test_shard_covers_members_once():
    for n in (1, 7, 256, 1000):
        for world in (1, 2, 3, 4, 8):
            owned = [m for r in range(world) for m in E.shard(n, world, r)]
            assert owned == list(range(n))
            sizes = [len(E.shard(n, world, r)) for r in range(world)]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        E.shard(4, 2, 2)


def test_member_factors_and_dt():
    prob, jf, kf, dt = E.member_problem(5)
    j, k = __import__("paper_1611_06721_b200.configs", fromlist=["x"]).ensemble_factors(256, 0)
    assert (jf, kf) == (float(j[5]), float(k[5]))
    assert abs(dt - 2.256829e-4 * kf) < 1e-18
    assert prob.kappa == 5e6 * kf


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = E.shard(10, world, rank)
        local = [E.MemberResult(m, 1.0, 1.0, 3, 1e-4, {"source": m}, float(m), 1.0 + rank)
                 for m in mine]
        allres = E.gather_results(local, dist)
        tmax = E.max_over_ranks(1.0 + rank, dist)
        q.put((rank, [r.member for r in allres], [r.iterations["source"] for r in allres], tmax))
    finally:
        dist.destroy_process_group()


def test_gather_and_max_over_ranks_gloo():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, members, payload, tmax in out:
        assert members == list(range(10))
        assert payload == list(range(10))
        assert tmax == 2.0
