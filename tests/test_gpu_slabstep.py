"""Sharded explicit step (BASELINE configs[4], ``slabstep.py`` +
``csrc/solver_slab.cuh``) against the oracle and the single-context device
loop.  With one GPU the ranks are emulated in one process: the slabs' phases
run one after another with the rank-order sums of the loopback communicator,
and every PCG solve is one cooperative launch whose CTA groups are the ranks
(the recipe's emulation — never separate launches that wait on one another).

Bars (north_star): A-field (a_c, a_n) within 1e-8 relative L2 of the oracle at
every step, every solve within +-1 iteration.
"""

from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

from oracle import mq_oracle as O
from tests.conftest import oracle_model

pytestmark = pytest.mark.gpu

REL_FIELD = 1e-8


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def _field(a_c, a_n):
    return np.concatenate([np.asarray(a_c), np.asarray(a_n)])


def _check_iters(it, tr, nsteps):
    src = np.array(tr.iters[O.FAM_SOURCE][1:]).reshape(nsteps, 2)
    assert np.max(np.abs(it[:, 0] - src[:, 0])) <= 1
    assert np.max(np.abs(it[:, 2] - src[:, 1])) <= 1
    assert np.max(np.abs(it[:, 1] - np.array(tr.iters[O.FAM_PREV]))) <= 1
    assert np.max(np.abs(it[:, 3] - np.array(tr.iters[O.FAM_CUR][1:]))) <= 1


@pytest.fixture(scope="module")
def oracle_c0_runs():
    spec, m = oracle_model(0)
    out = {}
    for strategy, n in (("cspe", 30), ("previous", 10)):
        out[strategy] = O.run(m, O.sinusoid(50.0), spec.dt, n, strategy=strategy, rel_tol=1e-8, max_cols=5)
    return spec, m, out


@pytest.mark.parametrize("world", [1, 2, 3, 4])
def test_sharded_step_config0_vs_oracle(gpu_ok, oracle_c0_runs, world):
    """Config 0, CSPE k = 5, 30 steps with recovery, 1-4 emulated ranks."""
    from paper_1611_06721_b200 import configs as C
    from paper_1611_06721_b200.slabstep import run_explicit_sharded
    spec, m, runs = oracle_c0_runs
    tr = runs["cspe"]
    n = 30
    res = run_explicit_sharded(C.make_problem(0), n, spec.dt, world=world, strategy="cspe", max_cols=5,
                               record_states=True)
    assert res.a_c_history.shape == (n, m.n_c) and res.a_n_history.shape == (n, m.n_n)
    worst = max(rel(_field(res.a_c_history[i], res.a_n_history[i]), _field(tr.a_c[i + 1], tr.a_n[i + 1]))
                for i in range(n))
    assert worst <= REL_FIELD, worst
    _check_iters(res.step_iterations, tr, n)
    # source family: one direction (every source rhs is a multiple of the
    # pattern, later inserts drop); coupling families full at k = 5 and evicting
    assert res.aggregates["basis_cols"] == [1, 5, 5]
    assert min(res.aggregates["evictions"][1:]) > 0


def test_sharded_step_previous_strategy(gpu_ok, oracle_c0_runs):
    from paper_1611_06721_b200 import configs as C
    from paper_1611_06721_b200.slabstep import run_explicit_sharded
    spec, m, runs = oracle_c0_runs
    tr = runs["previous"]
    n = 10
    res = run_explicit_sharded(C.make_problem(0), n, spec.dt, world=2, strategy="previous", record_states=True)
    worst = max(rel(_field(res.a_c_history[i], res.a_n_history[i]), _field(tr.a_c[i + 1], tr.a_n[i + 1]))
                for i in range(n))
    assert worst <= REL_FIELD, worst
    _check_iters(res.step_iterations, tr, n)


def test_sharded_conducting_block_is_bit_exact(gpu_ok):
    """The sharded K_cn^T a_c equals the single-context product (itself
    pinned bitwise to the reference) on every slab, and dt = 0 reproduces the
    state bit for bit through the owned-edge Euler update and the all-gather
    (schur.py:379-405)."""
    from paper_1611_06721_b200 import configs as C
    from paper_1611_06721_b200.device import DeviceGrid
    from paper_1611_06721_b200.slabstep import SlabStepper
    prob = C.make_problem(0)
    spec, m = oracle_model(0)
    a0 = np.random.default_rng(3).standard_normal(m.n_c) * 1e-3
    with DeviceGrid(prob) as g:
        w_ref = g.kcn_t_apply(a0)
    for world in (1, 3):
        st = SlabStepper(prob, world, strategy="zero")
        try:
            st.set_state(a0, 0.0)
            w = np.zeros(m.n_n)
            for s in st.slabs:
                s.rhs(1)
                w[s.gidx] = s.download(s.vecs["rhs_cpl"])
            assert np.array_equal(w, w_ref)
            st.step(0.0)
            assert np.array_equal(st.a_c, a0)
        finally:
            st.close()


@pytest.mark.slow
@pytest.mark.parametrize("world", [2, 4])
def test_sharded_step_config1_fields(gpu_ok, world):
    """64^3 (configs[1], Brauer iron, CSPE k = 5): the first 8 steps of the
    sharded step against the oracle fixture (per-step CountSketch of the
    A-field, tests/fieldcheck.py) and its iteration counts."""
    from paper_1611_06721_b200 import configs as C
    from paper_1611_06721_b200.slabstep import run_explicit_sharded
    from tests import fieldcheck as F
    ref = np.load(Path(__file__).parent / "golden" / "fields_cfg1_cspe.npz")
    dt = float(ref["dt"])
    n = 8
    res = run_explicit_sharded(C.make_problem(1), n, dt, world=world, strategy="cspe", max_cols=5,
                               record_states=True)
    n_c, n_n = int(ref["n_c"]), int(ref["n_n"])
    plan = F.sketch_plan(n_c + n_n)
    est = [F.sketched_rel(F.field_of(res.a_c_history[i], res.a_n_history[i]), ref["sketch"][i + 1],
                          ref["norm"][i + 1], plan) for i in range(n)]
    assert max(est) <= REL_FIELD, est
    it = res.step_iterations
    src = ref["iters_src"][1:].reshape(-1, 2)[:n]
    assert np.max(np.abs(it[:, 0] - src[:, 0])) <= 1 and np.max(np.abs(it[:, 2] - src[:, 1])) <= 1
    assert np.max(np.abs(it[:, 1] - ref["iters_prev"][:n])) <= 1
    assert np.max(np.abs(it[:, 3] - ref["iters_cur"][1:n + 1])) <= 1


@pytest.mark.slow
def test_sharded_step_128_matches_single_context(gpu_ok):
    """128^3 two-block geometry (configs[2]) with CSPE k = 5: 2 emulated ranks
    against the single-context device loop over 3 steps (A-field within 1e-8,
    iterations within +-1)."""
    from paper_1611_06721_b200 import configs as C
    from paper_1611_06721_b200 import PcgConfig, run_explicit
    from paper_1611_06721_b200.slabstep import run_explicit_sharded
    spec = C.config_spec(2)
    prob = C.make_problem(2)
    n = 3
    one = run_explicit(prob, t_end=n * spec.dt, dt=spec.dt, strategy="cspe", pcg=PcgConfig(rel_tol=1e-8),
                       max_cols=5, output_period=spec.dt * (1 - 1e-3), record_states=True)
    res = run_explicit_sharded(prob, n, spec.dt, world=2, strategy="cspe", max_cols=5, record_states=True)
    for i in range(n):
        e = rel(_field(res.a_c_history[i], res.a_n_history[i]), _field(one.a_c_history[i], one.a_n_history[i]))
        assert e <= REL_FIELD, (i, e)
    assert np.max(np.abs(res.step_iterations - one.step_iterations)) <= 1


def _two_gpu_worker(rank, world, port, q):
    import os

    import torch
    import torch.distributed as dist

    from paper_1611_06721_b200 import configs as C
    from paper_1611_06721_b200.slabstep import run_explicit_sharded
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        spec = C.config_spec(0)
        res = run_explicit_sharded(C.make_problem(0), 10, spec.dt, world=world, dist=dist, device=rank,
                                   strategy="cspe", max_cols=5, record_states=True)
        q.put((rank, res.step_iterations, res.a_c_history, res.a_n_history))
    finally:
        dist.destroy_process_group()


def test_sharded_step_two_processes(gpu_ok, oracle_c0_runs):
    """One rank per process and GPU (NCCL all-gathers, fused slab PCG over
    CUDA-IPC-mapped neighbour buffers).  Runs wherever two GPUs exist."""
    import socket

    import torch
    import torch.multiprocessing as mp
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs (one rank per GPU; ranks that wait on one another never share one)")
    spec, m, runs = oracle_c0_runs
    tr = runs["cspe"]
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_two_gpu_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted([q.get(timeout=300) for _ in procs], key=lambda o: o[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (_, it0, ac0, an0), (_, it1, ac1, an1) = out
    assert np.array_equal(it0, it1) and np.array_equal(ac0, ac1) and np.array_equal(an0, an1)
    for i in range(10):
        assert rel(_field(ac0[i], an0[i]), _field(tr.a_c[i + 1], tr.a_n[i + 1])) <= REL_FIELD


@pytest.mark.slow
def test_sharded_step_config4_grid_matches_single_context(gpu_ok):
    """configs[4] itself (256^3, Brauer, CSPE k = 5): the sharded step on 2
    emulated ranks against the single-context device loop over 2 steps with
    recovery (A-field within 1e-8 per step, every solve within +-1
    iteration).  No oracle run exists at 256^3 (hours of CPU); the
    single-context loop is the one pinned to the oracle at 16^3-128^3."""
    from paper_1611_06721_b200 import configs as C
    from paper_1611_06721_b200 import PcgConfig, run_explicit
    from paper_1611_06721_b200.slabstep import run_explicit_sharded
    spec = C.config_spec(4)
    prob = C.make_problem(4)
    n = 2
    one = run_explicit(prob, t_end=n * spec.dt, dt=spec.dt, strategy="cspe", pcg=PcgConfig(rel_tol=1e-8),
                       max_cols=5, output_period=spec.dt * (1 - 1e-3), record_states=True)
    res = run_explicit_sharded(prob, n, spec.dt, world=2, strategy="cspe", max_cols=5, record_states=True)
    for i in range(n):
        e = rel(_field(res.a_c_history[i], res.a_n_history[i]), _field(one.a_c_history[i], one.a_n_history[i]))
        assert e <= REL_FIELD, (i, e)
    assert np.max(np.abs(res.step_iterations - one.step_iterations)) <= 1
