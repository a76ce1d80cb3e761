"""configs[4] sharded explicit step (``slabstep.SlabStepper``): the host
sequence and the torch.distributed communicator at world size 2 over gloo on
CPU, with numpy slabs (tests/slabstep_numpy.py) standing in for the device
phases, against the single-domain oracle run (A-field within 1e-8 per step,
iterations within +-1)."""

from __future__ import annotations

import os
import socket

import numpy as np

NSTEPS = 6


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_1611_06721_b200 import configs as C
    from paper_1611_06721_b200.slabstep import SlabStepper, _Torch, run_explicit_sharded
    from tests.conftest import oracle_model
    from tests.slabstep_numpy import NumpySlabStep
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        spec, m = oracle_model(0)
        prob = C.make_problem(0)
        comm = _Torch(dist)
        # the communicator: rank-order sums, identical bits on every rank
        tot = comm.allreduce([np.array([0.1, 1e-17, 3.0]) * (rank + 1)])[0]
        sizes = comm.allgather([np.arange(rank + 2, dtype=np.float64)])
        st = SlabStepper(prob, world, dist=dist, strategy="cspe", max_cols=5, pcg="host", comm=comm,
                         slabs=[NumpySlabStep(m, rank, world, max_cols=5)])
        res = run_explicit_sharded(prob, NSTEPS, spec.dt, world=world, record_states=True, stepper=st)
        q.put((rank, tot, [s.size for s in sizes], res.step_iterations, res.a_c_history, res.a_n_history,
               st.diagnostics()["basis_cols"]))
    finally:
        dist.destroy_process_group()


def test_sharded_step_gloo_matches_oracle():
    import torch.multiprocessing as mp

    from oracle import mq_oracle as O
    from tests.conftest import oracle_model
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted([q.get(timeout=300) for _ in procs], key=lambda o: o[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    spec, m = oracle_model(0)
    tr = O.run(m, O.sinusoid(50.0), spec.dt, NSTEPS, strategy="cspe", rel_tol=1e-8, max_cols=5)
    (_, tot0, sz0, it0, ac0, an0, b0), (_, tot1, sz1, it1, ac1, an1, b1) = out
    assert np.array_equal(tot0, tot1) and np.array_equal(tot0, np.array([0.1, 1e-17, 3.0]) + np.array([0.2, 2e-17, 6.0]))
    assert sz0 == sz1 == [2, 3]
    # every rank took the same decisions and holds the same state
    assert np.array_equal(it0, it1) and np.array_equal(ac0, ac1) and np.array_equal(an0, an1) and b0 == b1
    for i in range(NSTEPS):
        f = np.concatenate([ac0[i], an0[i]])
        ref = np.concatenate([tr.a_c[i + 1], tr.a_n[i + 1]])
        assert np.linalg.norm(f - ref) <= 1e-8 * np.linalg.norm(ref), i
    src = np.array(tr.iters[O.FAM_SOURCE][1:]).reshape(NSTEPS, 2)
    assert np.max(np.abs(it0[:, 0] - src[:, 0])) <= 1 and np.max(np.abs(it0[:, 2] - src[:, 1])) <= 1
    assert np.max(np.abs(it0[:, 1] - np.array(tr.iters[O.FAM_PREV]))) <= 1
    assert np.max(np.abs(it0[:, 3] - np.array(tr.iters[O.FAM_CUR][1:]))) <= 1
