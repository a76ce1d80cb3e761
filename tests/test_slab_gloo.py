"""configs[4] i-slab decomposition: the distributed PCG host loop over
world-size-2 gloo with numpy slabs (CPU), against the single-domain oracle."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

from paper_1611_06721_b200.slab import slab_range


def test_slab_ranges():
    for nx in (8, 16, 256):
        for world in (1, 2, 3, 4, 8):
            if world > nx:
                continue
            rs = [slab_range(nx, world, r) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == nx
            assert all(a[1] == b[0] for a, b in zip(rs[:-1], rs[1:]))
    with pytest.raises(ValueError):
        slab_range(4, 5, 0)


def _model():
    from oracle import mq_oracle as O
    mat = np.zeros((12, 10, 9), np.int8)
    mat[4:8, 3:6, 3:6] = 1
    return O.assemble(mat, 0.1, O.Conductor(3e6, 0, 0, 500.0), [])


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, x0_given):
    import torch.distributed as dist

    from oracle import mq_oracle as O
    from paper_1611_06721_b200.slab import TorchComm, slab_pcg_solve
    from tests.slab_numpy import NumpySlab
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m = _model()
        inv = O.jacobi_inverse(m.kn.diagonal())[0]
        rng = np.random.default_rng(5)
        b = m.kn @ rng.standard_normal(m.n_n)
        x0 = rng.standard_normal(m.n_n) * 1e-2
        s = NumpySlab(m, rank, world, inv)
        s.set_global("b", b)
        if x0_given:
            s.set_global("x", x0)
        it, rel, conv, app = slab_pcg_solve([s], TorchComm(dist), x0_given=x0_given, rel_tol=1e-10)
        q.put((rank, it, rel, conv, app, s.own, s.own_values("x")))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("x0_given", [False, True])
def test_distributed_pcg_gloo_matches_single_domain(x0_given):
    import torch.multiprocessing as mp

    from oracle import mq_oracle as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, x0_given)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    m = _model()
    rng = np.random.default_rng(5)
    b = m.kn @ rng.standard_normal(m.n_n)
    x0 = rng.standard_normal(m.n_n) * 1e-2
    ref = O.pcg(m.kn_apply, b, x0=x0 if x0_given else None, rel_tol=1e-10,
                inv_diag=O.jacobi_inverse(m.kn.diagonal()))
    x = np.zeros(m.n_n)
    owned = np.zeros(m.n_n, dtype=int)
    its = set()
    for rank, it, rel, conv, app, own, xv in out:
        x[own] = xv
        owned[own] += 1
        its.add(it)
        assert conv and app == ref.applies
    assert np.all(owned == 1)                      # the slabs partition the dofs
    assert its == {ref.iterations}                 # every rank took the same decisions
    assert np.linalg.norm(x - ref.x) <= 1e-12 * np.linalg.norm(ref.x)


def _ipc_worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_1611_06721_b200.slab import IPC_HANDLE_BYTES, gather_ipc_tables
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = bytes([rank + 1]) * IPC_HANDLE_BYTES   # stand-in handle block
        handles, planes = gather_ipc_tables(mine, 10 + rank, dist)
        q.put((rank, [h[0] for h in handles], [len(h) for h in handles], planes))
    finally:
        dist.destroy_process_group()


def test_fused_peer_ipc_tables_gloo():
    """Host side of the fused slab kernel's setup: every rank ends up with all
    ranks' IPC handle blocks and plane counts in rank order."""
    import torch.multiprocessing as mp
    from paper_1611_06721_b200.slab import IPC_HANDLE_BYTES, gather_ipc_tables
    with pytest.raises(ValueError):
        gather_ipc_tables(b"x", 1)
    assert gather_ipc_tables(b"\0" * IPC_HANDLE_BYTES, 7) == ([b"\0" * IPC_HANDLE_BYTES], [7])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, first_bytes, sizes, planes in out:
        assert first_bytes == [1, 2, 3] and sizes == [IPC_HANDLE_BYTES] * 3 and planes == [10, 11, 12]
