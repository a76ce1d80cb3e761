"""Parity of the CUDA path (through the C ABI) against the pinned oracle.

Bars (BASELINE.json north_star): DoF numbering and masks bit-exact; A-field
within 1e-8 relative L2 per time step; PCG iteration counts within +-1.
Integer/structural results and the K_n SpMV (same CSR column order, no FMA)
must be bit-identical.
"""

from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

from oracle import mq_oracle as O
from tests.conftest import oracle_model

pytestmark = pytest.mark.gpu

REL_FIELD = 1e-8   # north_star: A-field (a_c, a_n) within 1e-8 relative L2 per step


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


@pytest.fixture(scope="module")
def c0(gpu_ok):
    from paper_1611_06721_b200 import configs as C
    from paper_1611_06721_b200.device import DeviceGrid
    spec, m = oracle_model(0)
    prob = C.make_problem(0)
    g = DeviceGrid(prob)
    yield spec, m, prob, g
    g.close()


def test_partition_and_masks_bit_exact(c0):
    spec, m, prob, g = c0
    nc, c = g.partition()
    assert (g.n_c, g.n_n) == (m.n_c, m.n_n) == (882, 9918)
    assert np.array_equal(nc, m.noncond_global)
    assert np.array_equal(c, m.cond_global)
    assert np.array_equal(g.mc_diag(), m.mc_diag)
    assert g.kn_diag == m.kn.diagonal()[0]
    assert g.kn_off == np.abs(m.kn.data).min()
    assert g.jacobi_inv == O.jacobi_inverse(m.kn.diagonal())[0]
    assert np.array_equal(prob.pattern, m.pattern)
    idx = g.noncond_index(m.noncond_global[[0, 5, -1]])
    assert list(idx) == [0, 5, m.n_n - 1]


def test_partition_two_blocks_and_boundary_cases(gpu_ok):
    """Disjoint blocks, a block touching the PEC boundary, a single cell."""
    from paper_1611_06721_b200.device import DeviceGrid, Problem
    N = 10
    cases = []
    mat = np.zeros((N, N, N), np.int8)
    mat[1:3, 2:5, 3:6] = 1
    mat[6:9, 5:8, 1:4] = 1
    cases.append(mat)
    mat = np.zeros((N, N, 7), np.int8)     # non-cubic, conductor on the boundary
    mat[0:3, 0:2, 0:7] = 1
    cases.append(mat)
    mat = np.zeros((4, 4, 4), np.int8)     # corner toy (tests/conftest.py:92-106)
    mat[0, 0, 0] = 1
    cases.append(mat)
    for mat in cases:
        m = O.assemble(mat, 0.1, O.Conductor(3e6, 0, 0, 500.0), [])
        g = DeviceGrid(Problem(material=mat, h=0.1, kappa=3e6, brauer=(0, 0, 500.0),
                               pattern=np.zeros(m.n_n)))
        nc, c = g.partition()
        assert np.array_equal(nc, m.noncond_global)
        assert np.array_equal(c, m.cond_global)
        assert np.array_equal(g.mc_diag(), m.mc_diag)
        x = np.random.default_rng(3).standard_normal(m.n_n)
        assert np.array_equal(g.kn_apply(x), m.kn @ x)
        xc = np.random.default_rng(4).standard_normal(m.n_c)
        assert np.array_equal(g.kcn_t_apply(xc), m.kcn.T @ xc)
        assert np.array_equal(g.kcn_apply(x), m.kcn @ x)
        g.close()


def test_kn_spmv_bitwise(c0, golden):
    spec, m, prob, g = c0
    rng = np.random.default_rng(20250819)
    x = rng.standard_normal(m.n_n)
    y = g.kn_apply(x)
    assert np.array_equal(y, golden["c0_spmv_y"])     # the reference's own scipy result
    for _ in range(3):
        x = rng.standard_normal(m.n_n) * rng.uniform(1e-6, 1e6)
        assert np.array_equal(g.kn_apply(x), m.kn @ x)


def test_conducting_block_products(c0, golden):
    spec, m, prob, g = c0
    st, xc = golden["c0b_kc_state"], golden["c0b_kc_x"]
    assert np.array_equal(g.kc_apply(st, xc), golden["c0_kc_y"])       # linear: bit-exact
    assert np.array_equal(g.kcn_t_apply(xc), golden["c0_kcnt_y"])
    x = np.random.default_rng(5).standard_normal(m.n_n)
    assert np.array_equal(g.kcn_apply(x), m.kcn @ x)


def test_brauer_kc_apply(gpu_ok, golden):
    from paper_1611_06721_b200 import configs as C
    from paper_1611_06721_b200.device import DeviceGrid
    prob = C.make_problem(0)
    prob.brauer = C.BRAUER_IRON
    with DeviceGrid(prob) as g:
        st, xc = golden["c0b_kc_state"], golden["c0b_kc_x"]
        y = g.kc_apply(st, xc)
        # exp() differs from numpy's by at most an ulp or two
        assert rel(y, golden["c0b_kc_y"]) <= 1e-14
        for scale in (0.0, 1e-3, 3e-3):   # up to deep saturation
            s = st * (scale / 2e-4) if scale else np.zeros_like(st)
            _, mb = oracle_model(0, brauer=C.BRAUER_IRON)
            assert rel(g.kc_apply(s, xc), mb.kc_apply(s, xc)) <= 1e-13


def test_pcg_matches_oracle(c0, golden):
    from paper_1611_06721_b200 import PcgConfig, Preconditioner, pcg_solve
    spec, m, prob, g = c0
    op = g.kn_operator()
    inv = O.jacobi_inverse(m.kn.diagonal())
    cfg = PcgConfig(rel_tol=1e-8, max_iter=5000, preconditioner=Preconditioner.JACOBI)
    rng = np.random.default_rng(7)
    b = m.kn @ rng.standard_normal(m.n_n)
    x0 = rng.standard_normal(m.n_n) * 1e-3
    for start in (None, x0, np.zeros(m.n_n)):
        x, rep = pcg_solve(op, b, x0=start, config=cfg)
        ref = O.pcg(m.kn_apply, b, x0=start, rel_tol=1e-8, inv_diag=inv)
        assert rep.converged and ref.converged
        assert abs(rep.iterations - ref.iterations) <= 1
        assert rep.applications == ref.applies
        assert rel(x, ref.x) <= 1e-8
        assert rep.final_rel_residual <= 1e-8


def test_pcg_semantics(c0):
    """krylov.py semantics: zero-iteration shortcut, zero rhs, budget, counts."""
    from paper_1611_06721_b200 import PcgConfig, Preconditioner, pcg_solve
    spec, m, prob, g = c0
    op = g.kn_operator()
    cfg = PcgConfig(rel_tol=1e-8, preconditioner=Preconditioner.JACOBI)
    # zero rhs, no x0: free (0 applications, rel 0)
    x, rep = pcg_solve(op, np.zeros(m.n_n), config=cfg)
    assert rep.iterations == 0 and rep.converged and rep.final_rel_residual == 0.0
    assert rep.applications == 0 and np.array_equal(x, np.zeros(m.n_n))
    # exact start vector: one application, x returned bit-identical
    xs = O.pcg(m.kn_apply, m.pattern, rel_tol=1e-12, inv_diag=O.jacobi_inverse(m.kn.diagonal())).x
    b = m.kn @ xs
    x, rep = pcg_solve(op, b, x0=xs, config=cfg)
    assert rep.iterations == 0 and rep.applications == 1 and np.array_equal(x, xs)
    # budget exhaustion: converged False with the last iterate
    x, rep = pcg_solve(op, m.pattern, config=PcgConfig(rel_tol=1e-14, max_iter=3,
                                                       preconditioner=Preconditioner.JACOBI))
    ref = O.pcg(m.kn_apply, m.pattern, rel_tol=1e-14, max_iter=3,
                inv_diag=O.jacobi_inverse(m.kn.diagonal()))
    assert not rep.converged and rep.iterations == 3 and not ref.converged
    assert rel(x, ref.x) <= 1e-12
    assert abs(rep.final_rel_residual - ref.rel) <= 1e-10 * ref.rel
    # no preconditioner
    x, rep = pcg_solve(op, m.pattern, config=PcgConfig(rel_tol=1e-8))
    ref = O.pcg(m.kn_apply, m.pattern, rel_tol=1e-8)
    assert abs(rep.iterations - ref.iterations) <= 1 and rel(x, ref.x) <= 1e-8
    # non-finite input rejected like sparse.as_vector
    bad = m.pattern.copy()
    bad[3] = np.nan
    with pytest.raises(ValueError):
        pcg_solve(op, bad, config=cfg)


def test_csr_path_reference_cases(gpu_ok):
    """The reference's krylov tests, through the general CSR device path."""
    import scipy.sparse as sp

    from paper_1611_06721_b200 import (IndefiniteOperatorError, JacobiPreconditioner,
                                       PcgConfig, Preconditioner, pcg_solve)
    rng = np.random.default_rng(20250819)
    b = rng.standard_normal(5)
    x, rep = pcg_solve(sp.identity(5, format="csr"), b)
    assert rep.converged and rep.iterations == 1 and np.allclose(x, b, rtol=0, atol=1e-14)
    q = np.linalg.qr(rng.standard_normal((30, 30)))[0]
    dense = (q * rng.uniform(0.5, 50.0, 30)) @ q.T
    dense = 0.5 * (dense + dense.T)
    b = rng.standard_normal(30)
    for kind in (Preconditioner.NONE, Preconditioner.JACOBI):
        x, rep = pcg_solve(dense, b, config=PcgConfig(rel_tol=1e-10, max_iter=200,
                                                     preconditioner=kind))
        ref = O.pcg(lambda v: sp.csr_matrix(dense) @ v, b, rel_tol=1e-10, max_iter=200,
                    inv_diag=O.jacobi_inverse(np.diag(dense)) if kind is Preconditioner.JACOBI else None)
        assert rep.converged and abs(rep.iterations - ref.iterations) <= 1
        assert np.linalg.norm(dense @ x - b) / np.linalg.norm(b) <= 1e-8
    lap = np.array([[1.0, -1, 0, 0], [-1, 2, -1, 0], [0, -1, 2, -1], [0, 0, -1, 1]])
    bb = np.array([1.0, -0.5, 0.25, -0.75])
    x, rep = pcg_solve(lap, bb, x0=np.zeros(4), config=PcgConfig(rel_tol=1e-12, max_iter=100))
    assert rep.converged and np.allclose(x, np.linalg.pinv(lap) @ bb, rtol=0, atol=1e-8)
    with pytest.raises(IndefiniteOperatorError):
        pcg_solve(np.diag([1.0, -1.0]), np.array([1.0, 1.0]))
    x, rep = pcg_solve(np.diag([2.0, 2.0]), np.array([2.0, 4.0]),
                       config=PcgConfig(preconditioner=Preconditioner.JACOBI),
                       preconditioner=JacobiPreconditioner(np.full(2, 2.0)))
    assert rep.converged and np.allclose(x, [1.0, 2.0], rtol=0, atol=1e-12)
    with pytest.raises(TypeError):
        pcg_solve(lambda v: v, np.ones(2))


def test_csr_path_on_assembled_kn(c0):
    """An externally supplied CSR K_n (non-FIT models) on
    the general CSR device PCG: the configs[0] matrix as scipy CSR against
    the matrix-free stencil path and the oracle."""
    import scipy.sparse as sp

    from paper_1611_06721_b200 import PcgConfig, Preconditioner, pcg_solve
    spec, m, prob, g = c0
    cfg = PcgConfig(rel_tol=1e-8, preconditioner=Preconditioner.JACOBI)
    x_csr, rep_csr = pcg_solve(sp.csr_matrix(m.kn), m.pattern, config=cfg)
    x_st, rep_st = pcg_solve(g.kn_operator(), m.pattern, config=cfg)
    ref = O.pcg(m.kn_apply, m.pattern, rel_tol=1e-8, inv_diag=O.jacobi_inverse(m.kn.diagonal()))
    assert rep_csr.converged and abs(rep_csr.iterations - ref.iterations) <= 1
    assert rel(x_csr, ref.x) <= 1e-8 and rel(x_csr, x_st) <= 1e-8


def test_cspe_strategy_parity(c0, golden):
    from paper_1611_06721_b200 import DeviceStrategy, RhsFamily
    spec, m, prob, g = c0
    inv = O.jacobi_inverse(m.kn.diagonal())
    rng = np.random.default_rng(11)
    seq = [O.pcg(m.kn_apply, m.kn @ rng.standard_normal(m.n_n), rel_tol=1e-8, inv_diag=inv).x
           for _ in range(6)]
    seq.append(seq[2] * 3.0)      # dependent -> dropped
    seq.append(np.zeros(m.n_n))   # zero -> dropped
    strat = DeviceStrategy(g, "cspe", max_cols=5, drop_tol=1e-8)
    cache = O.SpeCache(m.n_n, m.kn_apply, max_cols=5, drop_tol=1e-8)
    fam = RhsFamily.SOURCE_CURRENT
    rhs = m.kn @ rng.standard_normal(m.n_n)
    assert np.array_equal(strat.start_vector(fam, rhs), np.zeros(m.n_n))  # empty cache
    for v in seq:
        strat.observe(fam, v)
        cache.insert(v)
        assert strat.basis_size(fam) == cache.k
        assert strat.basis_size(RhsFamily.COUPLING_FROM_PREVIOUS_STATE) == 0
    assert strat.maintenance_applies == cache.products
    U, KU, G = strat.cache_export(fam)
    assert rel(G, cache.G) <= 1e-10
    assert np.max(np.abs(U - cache.U)) <= 1e-10 * np.max(np.abs(cache.U))
    assert rel(KU, cache.KU) <= 1e-10
    x0 = strat.start_vector(fam, rhs)
    assert rel(x0, cache.project(rhs)) <= 1e-8
    # family isolation
    assert np.array_equal(strat.start_vector(RhsFamily.COUPLING_FROM_CURRENT_STATE, rhs),
                          np.zeros(m.n_n))


def test_pod_strategy_parity(c0):
    from paper_1611_06721_b200 import DeviceStrategy, RhsFamily
    spec, m, prob, g = c0
    inv = O.jacobi_inverse(m.kn.diagonal())
    rng = np.random.default_rng(12)
    seq = [O.pcg(m.kn_apply, m.kn @ rng.standard_normal(m.n_n), rel_tol=1e-8, inv_diag=inv).x
           for _ in range(5)]
    seq += [seq[0] + 1e-3 * seq[1], seq[3] * 0.5, seq[1] - 1e-6 * seq[2]]
    strat = DeviceStrategy(g, "pod", n_pod=6, eps_pod=1e-4)
    snap = O.Snapshots(m.n_n, n_pod=6, eps_pod=1e-4)
    pod = O.PodStrategyOracle(m.n_n, m.kn_apply, n_pod=6, eps_pod=1e-4)
    fam = RhsFamily.COUPLING_FROM_PREVIOUS_STATE
    rhs = m.kn @ rng.standard_normal(m.n_n)
    for i, v in enumerate(seq):
        strat.observe(fam, v)
        pod.observe(O.FAM_PREV, v)
        x_dev = strat.start_vector(fam, rhs)
        x_ref = pod.start(O.FAM_PREV, rhs)
        d = strat.diagnostics()
        assert d["pod_k"] == pod.last_k, i
        # info = sum(sigma_k)/sum(sigma): the dropped modes sit at the
        # round-off floor (sigma ~ 1e-8 sigma_1), where LAPACK and the device
        # Jacobi solver legitimately disagree at ~1e-9
        assert abs(d["pod_info"] - pod.last_info) <= 1e-7
        assert d["maintenance_applies"] == pod.applies
        assert rel(x_dev, x_ref) <= 1e-8, i
    assert abs(strat.diagnostics()["min_pod_info"] - pod.min_info) <= 1e-7


def test_strategy_edge_cases(c0):
    """startvec.py edge cases the reference tests (test_startvec.py: zero and
    non-finite columns, rank-one and all-zero snapshot buffers, empty
    buffers): device strategies vs the oracle's."""
    from paper_1611_06721_b200 import DeviceStrategy, RhsFamily
    spec, m, prob, g = c0
    inv = O.jacobi_inverse(m.kn.diagonal())
    rng = np.random.default_rng(21)
    rhs = m.kn @ rng.standard_normal(m.n_n)
    v = O.pcg(m.kn_apply, m.kn @ rng.standard_normal(m.n_n), rel_tol=1e-8, inv_diag=inv).x
    fam = RhsFamily.SOURCE_CURRENT
    # CSPE: zero / non-finite columns are dropped, the cache is unchanged
    strat = DeviceStrategy(g, "cspe", max_cols=3, drop_tol=1e-8)
    cache = O.SpeCache(m.n_n, m.kn_apply, max_cols=3, drop_tol=1e-8)
    bad = v.copy()
    bad[7] = np.nan
    for col in (np.zeros(m.n_n), v, bad, v * np.inf):
        strat.observe(fam, col)
        cache.insert(col)
        assert strat.basis_size(fam) == cache.k
    assert strat.maintenance_applies == cache.products == 1
    assert rel(strat.start_vector(fam, rhs), cache.project(rhs)) <= 1e-8
    # POD: empty buffer -> zero start; all-zero snapshots -> zero start, k = 0
    pstrat = DeviceStrategy(g, "pod", n_pod=4, eps_pod=1e-4)
    pod = O.PodStrategyOracle(m.n_n, m.kn_apply, n_pod=4, eps_pod=1e-4)
    assert np.array_equal(pstrat.start_vector(fam, rhs), np.zeros(m.n_n))
    for _ in range(2):
        pstrat.observe(fam, np.zeros(m.n_n))
        pod.observe(O.FAM_SOURCE, np.zeros(m.n_n))
    x_dev, x_ref = pstrat.start_vector(fam, rhs), pod.start(O.FAM_SOURCE, rhs)
    assert np.array_equal(x_dev, np.zeros(m.n_n)) and np.array_equal(x_ref, np.zeros(m.n_n))
    assert pstrat.diagnostics()["pod_k"] == pod.last_k == 0
    # rank-one snapshots: one retained mode, start = its Galerkin projection
    pstrat = DeviceStrategy(g, "pod", n_pod=4, eps_pod=1e-4)
    pod = O.PodStrategyOracle(m.n_n, m.kn_apply, n_pod=4, eps_pod=1e-4)
    for a in (1.0, -2.0, 0.5, 3.0, 4.0):  # more than n_pod: the ring wraps
        pstrat.observe(fam, a * v)
        pod.observe(O.FAM_SOURCE, a * v)
    x_dev, x_ref = pstrat.start_vector(fam, rhs), pod.start(O.FAM_SOURCE, rhs)
    assert pstrat.diagnostics()["pod_k"] == pod.last_k == 1
    assert rel(x_dev, x_ref) <= 1e-8


@pytest.mark.parametrize("strategy,nsteps", [("cspe", 100), ("pod", 30), ("previous", 30)])
def test_transient_config0_device_loop(gpu_ok, strategy, nsteps):
    """run_explicit twin (device-resident loop, CUDA graph replay) vs oracle."""
    from paper_1611_06721_b200 import configs as C
    from paper_1611_06721_b200 import PcgConfig, run_explicit
    spec, m = oracle_model(0)
    prob = C.make_problem(0)
    tr = O.run(m, O.sinusoid(50.0), spec.dt, nsteps, strategy=strategy, rel_tol=1e-8,
               max_cols=5, n_pod=20, eps_pod=1e-4)
    res = run_explicit(prob, t_end=nsteps * spec.dt, dt=spec.dt, strategy=strategy,
                       pcg=PcgConfig(rel_tol=1e-8, max_iter=5000),
                       output_period=spec.dt * (1 - 1e-3), max_cols=5, n_pod=20,
                       eps_pod=1e-4, record_states=True, use_graph=False)
    hist = res.a_c_history
    assert hist.shape == (nsteps, m.n_c) and res.a_n_history.shape == (nsteps, m.n_n)
    # the north-star bar: the whole A-field (a_c, a_n) at every step
    worst = max(rel(np.concatenate([hist[i], res.a_n_history[i]]),
                    np.concatenate([tr.a_c[i + 1], tr.a_n[i + 1]])) for i in range(nsteps))
    assert worst <= REL_FIELD, worst
    assert max(rel(hist[i], tr.a_c[i + 1]) for i in range(nsteps)) <= REL_FIELD
    it = res.step_iterations
    src = np.array(tr.iters[O.FAM_SOURCE][1:]).reshape(nsteps, 2)
    assert np.max(np.abs(it[:, 0] - src[:, 0])) <= 1
    assert np.max(np.abs(it[:, 2] - src[:, 1])) <= 1
    assert np.max(np.abs(it[:, 1] - np.array(tr.iters[O.FAM_PREV]))) <= 1
    assert np.max(np.abs(it[:, 3] - np.array(tr.iters[O.FAM_CUR][1:]))) <= 1
    assert np.array_equal(res.final_a_n, res.a_n_history[-1])
    # graph replay gives the same trajectory as eager launches
    res_g = run_explicit(prob, t_end=nsteps * spec.dt, dt=spec.dt, strategy=strategy,
                         pcg=PcgConfig(rel_tol=1e-8, max_iter=5000),
                         output_period=spec.dt * (1 - 1e-3), max_cols=5, n_pod=20,
                         eps_pod=1e-4, use_graph=True)
    assert np.array_equal(res_g.final_a_c, hist[-1])
    assert np.array_equal(res_g.step_iterations, it)


@pytest.mark.parametrize("index", [0, 2])
def test_device_probe_bitwise_vs_reference(gpu_ok, golden, index):
    """mq_probe_b (model.py:415-425) on the reference's own probe states:
    b2 in the reference's operation order and numpy's pairwise mean give the
    reference's value bit for bit."""
    from pathlib import Path
    from tests.golden.make_golden_probe import probe_states
    from paper_1611_06721_b200 import configs as C
    from paper_1611_06721_b200 import SchurOperator
    ref = np.load(Path(__file__).parent / "golden" / "reference_probe.npz")
    op = SchurOperator(C.make_problem(index), strategy="previous")
    cells = op.set_probe()
    assert np.array_equal(cells, ref[f"c{index}_probe_cells"])
    vals = [op.probe_b(a_c) for a_c, _ in probe_states(index, op.grid.n_c, op.grid.n_n, golden)]
    assert np.array_equal(np.array(vals), ref[f"c{index}_probe_values"])
    with pytest.raises(Exception):
        op.set_probe(np.array([0], dtype=np.int64))   # an air cell


def test_device_probe_in_run(gpu_ok):
    """run_explicit(probe="device"): B_probe logged inside the step graph
    equals the oracle's probe of its own trajectory within the field bar."""
    from paper_1611_06721_b200 import configs as C
    from paper_1611_06721_b200 import PcgConfig, run_explicit
    spec, m = oracle_model(0)
    nsteps = 20
    tr = O.run(m, O.sinusoid(50.0), spec.dt, nsteps, strategy="cspe", rel_tol=1e-8, max_cols=5)
    cells = O.default_probe_cells(m, (spec.N,) * 3)
    ref_b = np.array([O.probe_b(m, O.full_interior(m, a, b), cells)
                      for a, b in zip(tr.a_c, tr.a_n)])
    for use_graph in (False, True):
        res = run_explicit(C.make_problem(0), t_end=nsteps * spec.dt, dt=spec.dt, strategy="cspe",
                           pcg=PcgConfig(rel_tol=1e-8), output_period=spec.dt * (1 - 1e-3),
                           max_cols=5, probe="device", use_graph=use_graph)
        b = res.probe_b
        assert b.shape == (nsteps + 1,)
        assert np.max(np.abs(b - ref_b) / np.abs(ref_b).max()) <= REL_FIELD
    # segmented loop (outputs every 2nd step) probes the same states
    res2 = run_explicit(C.make_problem(0), t_end=nsteps * spec.dt, dt=spec.dt, strategy="cspe",
                        pcg=PcgConfig(rel_tol=1e-8), output_period=2 * spec.dt * (1 - 1e-3),
                        max_cols=5, probe="device")
    assert np.max(np.abs(res2.probe_b - ref_b[::2]) / np.abs(ref_b).max()) <= REL_FIELD


def test_schur_loop_semantics(gpu_ok):
    """test_schur.py cases on the device loop: a zero source from a zero state
    stays exactly zero with zero iterations; the final state does not depend
    on the start-vector strategy; output rows, validation and the step
    budget; a non-finite state names the failing step."""
    from paper_1611_06721_b200 import configs as C
    from paper_1611_06721_b200 import PcgConfig, SchurOperator, StepFailureError, run_explicit
    from paper_1611_06721_b200.schur import explicit_euler_step
    spec, m = oracle_model(0)
    quiet = C.make_problem(0)
    quiet.pattern = np.zeros_like(quiet.pattern)
    res = run_explicit(quiet, t_end=5 * spec.dt, dt=spec.dt, strategy="previous",
                       pcg=PcgConfig(rel_tol=1e-8))
    assert not res.final_a_c.any() and not res.final_a_n.any()
    assert res.aggregates["iterations"] == {"source": 0, "coupling_current": 0, "coupling_previous": 0}
    finals = {}
    for strategy in ("previous", "cspe", "pod", "zero"):
        finals[strategy] = run_explicit(C.make_problem(0), t_end=12 * spec.dt, dt=spec.dt, strategy=strategy,
                                        pcg=PcgConfig(rel_tol=1e-10), max_cols=5, n_pod=6).final_a_c
    for strategy in ("cspe", "pod", "zero"):
        assert rel(finals[strategy], finals["previous"]) <= 1e-8, strategy
    res = run_explicit(C.make_problem(0), t_end=10 * spec.dt, dt=spec.dt, strategy="cspe",
                       pcg=PcgConfig(rel_tol=1e-8), max_cols=5, output_period=2 * spec.dt, probe="device")
    assert res.times[0] == 0.0 and res.times[-1] == pytest.approx(10 * spec.dt, rel=1e-12)
    assert np.all(np.diff(res.times) > 0) and len(res.times) == len(res.probe_b) == 6
    assert res.aggregates["steps"] == 10 and res.aggregates["solves"]["source"] >= 10
    prob = C.make_problem(0)
    for kw in ({"t_end": 0.0, "dt": spec.dt}, {"t_end": 1.0, "dt": "sideways"}, {"t_end": 1.0, "dt": -1e-3},
               {"t_end": 1.0, "dt": spec.dt, "output_period": 0.0}):
        with pytest.raises(ValueError):
            run_explicit(prob, **kw)
    with pytest.raises(StepFailureError):
        run_explicit(prob, t_end=1.0, dt=1e-6, strategy="previous", max_steps=10)
    op = SchurOperator(C.make_problem(0), pcg=PcgConfig(rel_tol=1e-8), strategy="previous")
    with pytest.raises(StepFailureError, match="7"):
        explicit_euler_step((np.full(m.n_c, 1e300), 0.0), 1e9, op, step_index=7)


def test_auto_dt_reestimation(gpu_ok):
    """dt="auto" re-estimates every reestimate_every steps (schur.py:548-557):
    with linear iron the bound does not move, so the run equals the one with
    a single estimate bit for bit and counts its refreshes."""
    from paper_1611_06721_b200 import configs as C
    from paper_1611_06721_b200 import PcgConfig, run_explicit
    spec, m = oracle_model(0)
    kw = dict(strategy="cspe", pcg=PcgConfig(rel_tol=1e-8), max_cols=5, power_iters=60)
    once = run_explicit(C.make_problem(0), t_end=8.5 * spec.dt, dt="auto", reestimate_every=0,
                        output_period=spec.dt * (1 - 1e-3), **kw)
    again = run_explicit(C.make_problem(0), t_end=8.5 * spec.dt, dt="auto", reestimate_every=3,
                         output_period=spec.dt * (1 - 1e-3), **kw)
    assert once.aggregates["steps"] == again.aggregates["steps"] == 9
    assert once.aggregates["cfl_refreshes"] == 0 and again.aggregates["cfl_refreshes"] == 2
    assert again.aggregates["dt"] == once.aggregates["dt"]
    assert np.array_equal(again.final_a_c, once.final_a_c)
    assert np.array_equal(again.times, once.times)


def test_trace_csv_deterministic(gpu_ok):
    """The reference's trace CSV (bench.py:341-357) from two identical device
    runs is byte-identical (test_bench.py: test_benchmark_is_deterministic)."""
    from paper_1611_06721_b200 import configs as C
    from paper_1611_06721_b200 import PcgConfig, run_explicit
    from paper_1611_06721_b200.schur import TRACE_HEADER, trace_bytes
    spec, m = oracle_model(0)
    runs = [run_explicit(C.make_problem(0), t_end=6 * spec.dt, dt=spec.dt, strategy=strat,
                         pcg=PcgConfig(rel_tol=1e-8), max_cols=5, n_pod=6, probe="device",
                         output_period=2 * spec.dt * (1 - 1e-3))
            for strat in ("pod", "pod")]
    a, b = (trace_bytes(r) for r in runs)
    assert a == b
    lines = a.decode().splitlines()
    assert lines[0] == TRACE_HEADER and len(lines) == 1 + runs[0].n_rows == 5


TRACE_RUNS = [("cspe", 100, 1), ("pod", 30, 1), ("previous", 30, 1), ("cspe", 30, 3), ("pod", 30, 3)]


@pytest.mark.parametrize("strategy,nsteps,every", TRACE_RUNS)
def test_trace_rows_match_reference(gpu_ok, strategy, nsteps, every):
    """Every trace row of the device loop against the REFERENCE's own
    run_explicit on config 0 (tests/golden/reference_trace.npz, made by
    make_golden_trace.py with the reference's B probe): times bit-exact;
    basis_cols (schur.py:533), pod_k (window max, :535) and pod_info (window
    min of the strategy's last_info, :536) exact; the per-row iteration means
    within +-1; B_probe within the field bar.  (The whole CSV cannot be
    byte-identical: B_probe of a trajectory that differs from the reference's
    at the 1e-9 level differs in its last digits.)  Output every step runs the
    device-resident loop with the device diagnostics log; every third step runs
    the segmented loop (windows of three Euler steps)."""
    from paper_1611_06721_b200 import configs as C
    from paper_1611_06721_b200 import PcgConfig, run_explicit
    from paper_1611_06721_b200.schur import trace_bytes
    g = np.load(Path(__file__).parent / "golden" / "reference_trace.npz")
    key = f"{strategy}_{nsteps}_{every}"
    dt = float(g["dt"])
    res = run_explicit(C.make_problem(0), t_end=nsteps * dt, dt=dt, strategy=strategy,
                       pcg=PcgConfig(rel_tol=1e-8, max_iter=5000),
                       output_period=every * dt * (1 - 1e-3), probe="device", max_cols=5, n_pod=20,
                       eps_pod=1e-4)
    assert res.n_rows == g[f"{key}_times"].size
    assert np.array_equal(res.times, g[f"{key}_times"])
    assert np.array_equal(res.basis_cols, g[f"{key}_basis_cols"]), (res.basis_cols, g[f"{key}_basis_cols"])
    assert np.array_equal(res.pod_k, g[f"{key}_pod_k"]), (res.pod_k, g[f"{key}_pod_k"])
    ref_info = g[f"{key}_pod_info"]
    assert np.all((res.pod_info == 1.0) == (ref_info == 1.0))
    # info = sum(sigma_<=k) / sum(sigma): each singular value of snapshots
    # that differ by ~1e-8 relative (the field bar) moves by ~1e-8 sigma_1
    info_tol = 20 * REL_FIELD
    assert np.max(np.abs(res.pod_info - ref_info)) <= info_tol, np.max(np.abs(res.pod_info - ref_info))
    for col in ("iters_src", "iters_cpl_prev", "iters_cpl_cur"):
        assert np.max(np.abs(getattr(res, col) - g[f"{key}_{col}"])) <= 1.0, col
    b_ref = g[f"{key}_probe_b"]
    assert np.max(np.abs(res.probe_b - b_ref)) <= REL_FIELD * np.abs(b_ref).max()
    agg = g[f"{key}_agg"]
    assert res.aggregates["steps"] == int(agg[0])
    assert res.aggregates["max_basis_cols"] == int(agg[4])
    assert abs(res.aggregates["min_pod_info"] - agg[3]) <= info_tol
    lines, ref_lines = trace_bytes(res).decode().splitlines(), bytes(g[f"{key}_trace"]).decode().splitlines()
    assert lines[0] == ref_lines[0] and len(lines) == len(ref_lines)
    for a, b in zip(lines[1:], ref_lines[1:]):
        fa, fb = a.split(","), b.split(",")
        assert fa[0] == fb[0] and fa[5:7] == fb[5:7]   # t, basis_cols, pod_k: identical text


def test_single_step_api_matches_oracle(gpu_ok):
    """explicit_euler_step / recover_an / SchurOperator.solve_kn twins."""
    from paper_1611_06721_b200 import configs as C
    from paper_1611_06721_b200 import (PcgConfig, RhsFamily, SchurOperator,
                                       explicit_euler_step, recover_an)
    spec, m = oracle_model(0)
    prob = C.make_problem(0)
    op = SchurOperator(prob, pcg=PcgConfig(rel_tol=1e-8), strategy="cspe", max_cols=5)
    ref = O.SchurOracle(m, O.sinusoid(50.0), "cspe", 1e-8, 5000, 5)
    a, a_ref, t = np.zeros(m.n_c), np.zeros(m.n_c), 0.0
    an, (r1, r2) = recover_an(op, a, t)
    an_ref, (q1, q2) = ref.recover(a_ref, t)
    assert rel(an, an_ref) <= REL_FIELD
    for step in range(1, 6):
        a, (r1, r2) = explicit_euler_step((a, t), spec.dt, op, step_index=step)
        a_ref, (q1, q2) = ref.euler(a_ref, t, spec.dt, step)
        t += spec.dt
        assert abs(r1.iterations - q1.iterations) <= 1 and abs(r2.iterations - q2.iterations) <= 1
        assert rel(a, a_ref) <= REL_FIELD
        an, _ = recover_an(op, a, t)
        an_ref, _ = ref.recover(a_ref, t)
        assert rel(an, an_ref) <= REL_FIELD
    assert op.solve_count(RhsFamily.SOURCE_CURRENT) == 11
    # dt = 0 reproduces the state bit for bit (schur.py:386-387)
    a2, _ = explicit_euler_step((a, t), 0.0, op)
    assert np.array_equal(a2, a)
    with pytest.raises(ValueError):
        explicit_euler_step((a, t), -1.0, op)


@pytest.mark.slow
def test_config1_first_steps(gpu_ok, golden):
    """64^3 Brauer: first two steps against the reference's own numbers."""
    from paper_1611_06721_b200 import configs as C
    from paper_1611_06721_b200 import PcgConfig, run_explicit
    spec = C.config_spec(1)
    prob = C.make_problem(1)
    res = run_explicit(prob, t_end=2 * spec.dt, dt=spec.dt, strategy="cspe",
                       pcg=PcgConfig(rel_tol=1e-8), output_period=spec.dt * (1 - 1e-3),
                       max_cols=5, record_states=True)
    norms = np.linalg.norm(res.a_c_history, axis=1)
    ref = golden["c1_run_cspe_a_c_norms"][1:]
    assert np.all(np.abs(norms - ref) <= REL_FIELD * ref)
    it = golden["c1_run_cspe_iters"]
    assert np.max(np.abs(res.step_iterations[:, 3] - it[1:, 2])) <= 1
    assert np.max(np.abs(res.step_iterations[:, 1] - it[1:, 1])) <= 1


@pytest.mark.slow
def test_overlapped_source_update(gpu_ok, monkeypatch):
    """64^3 (resident PCG kernel): the source family's cache update on the
    side stream (its reductions run on the idle SMs' smaller grid, so the
    summation tree differs) is deterministic — graph replay and eager
    launches agree bit for bit — and stays within the field bar of the
    serial order."""
    from paper_1611_06721_b200 import configs as C
    from paper_1611_06721_b200 import PcgConfig, run_explicit
    spec = C.config_spec(1)
    runs = {}
    for ov in ("0", "1"):
        monkeypatch.setenv("MQ_OVERLAP", ov)
        for graph in (True, False):
            runs[ov, graph] = run_explicit(C.make_problem(1), t_end=12 * spec.dt, dt=spec.dt, strategy="cspe",
                                           pcg=PcgConfig(rel_tol=1e-8), max_cols=5,
                                           output_period=spec.dt * (1 - 1e-3), use_graph=graph)
    for ov in ("0", "1"):
        assert np.array_equal(runs[ov, True].final_a_c, runs[ov, False].final_a_c), ov
        assert np.array_equal(runs[ov, True].step_iterations, runs[ov, False].step_iterations), ov
    assert rel(runs["1", True].final_a_c, runs["0", True].final_a_c) <= REL_FIELD
    assert np.max(np.abs(runs["1", True].step_iterations - runs["0", True].step_iterations)) <= 1
    # every insert happened (the deferred one of the last recovery included)
    ag1, ag0 = runs["1", True].aggregates, runs["0", True].aggregates
    assert ag1["maintenance_applies"] == ag0["maintenance_applies"]
    assert abs(ag1["pcg_applies"] - ag0["pcg_applies"]) <= 4 * ag0["steps"]   # +-1 per solve
    assert np.array_equal(runs["1", True].basis_cols, runs["0", True].basis_cols)


@pytest.mark.parametrize("strategy", ["cspe", "pod"])
def test_step_graph_under_barrier_stress(gpu_ok, strategy, monkeypatch):
    """64^3 step graphs (resident PCG on the main stream, cache updates forked
    onto the side stream under it, deferred inserts) with the PCG kernels'
    CTAs delayed after every grid barrier (MQ_PCG_STRESS): the side-stream
    work now overlaps different parts of the solves, yet the trajectory,
    iteration counts and basis sizes are bit-identical to the unstressed run
    (the fork/join edges order every shared buffer)."""
    from paper_1611_06721_b200 import configs as C
    from paper_1611_06721_b200 import PcgConfig, run_explicit
    spec = C.config_spec(1)
    runs = []
    for stress in (None, "20000"):
        if stress:
            monkeypatch.setenv("MQ_PCG_STRESS", stress)
        else:
            monkeypatch.delenv("MQ_PCG_STRESS", raising=False)
        runs.append(run_explicit(C.make_problem(1), t_end=6 * spec.dt, dt=spec.dt, strategy=strategy,
                                 pcg=PcgConfig(rel_tol=1e-8), max_cols=5, n_pod=20,
                                 output_period=spec.dt * (1 - 1e-3)))
    assert np.array_equal(runs[0].final_a_c, runs[1].final_a_c)
    assert np.array_equal(runs[0].final_a_n, runs[1].final_a_n)
    assert np.array_equal(runs[0].step_iterations, runs[1].step_iterations)
    assert np.array_equal(runs[0].basis_cols, runs[1].basis_cols)
    assert np.array_equal(runs[0].pod_k, runs[1].pod_k)


@pytest.mark.slow
def test_host_step_api_matches_device_loop(gpu_ok):
    """64^3: explicit_euler_step + recover_an from the host (each call leaves
    its coupling-family insert pending on the device for the next call's side
    stream) reproduce the device-resident loop bit for bit, and every insert
    is accounted for."""
    from paper_1611_06721_b200 import configs as C
    from paper_1611_06721_b200 import PcgConfig, SchurOperator, explicit_euler_step, recover_an, run_explicit
    from paper_1611_06721_b200.schur import step_times
    spec = C.config_spec(1)
    n = 6
    res = run_explicit(C.make_problem(1), t_end=n * spec.dt, dt=spec.dt, strategy="cspe",
                       pcg=PcgConfig(rel_tol=1e-8), max_cols=5, output_period=spec.dt * (1 - 1e-3))
    dts, _ = step_times(n * spec.dt, spec.dt, spec.dt * (1 - 1e-3))   # the loop's own step sizes
    assert len(dts) == n
    op = SchurOperator(C.make_problem(1), pcg=PcgConfig(rel_tol=1e-8), strategy="cspe", max_cols=5)
    a, t = np.zeros(op.grid.n_c), 0.0
    recover_an(op, a, t)
    its = []
    for s, dt in enumerate(dts):
        a, (r1, r2) = explicit_euler_step((a, t), dt, op, s + 1)
        t += dt
        a_n, (q1, q2) = recover_an(op, a, t)
        its.append([r1.iterations, r2.iterations, q1.iterations, q2.iterations])
    assert np.array_equal(np.asarray(its), res.step_iterations)
    assert np.array_equal(a, res.final_a_c)
    assert np.array_equal(a_n, res.final_a_n)
    d = op.diagnostics()
    assert d.maintenance_applies == res.aggregates["maintenance_applies"]
    assert d.pcg_applies == res.aggregates["pcg_applies"]
    op.grid.close()


def test_probe_after_host_calls(gpu_ok):
    """probe_b() after a host recovery call returns the value that call
    computed with its results (no device round trip); after an Euler call,
    a state upload or new probe cells it is computed afresh.  Every value
    equals probe_b(state) on the same state bit for bit."""
    from paper_1611_06721_b200 import configs as C
    from paper_1611_06721_b200 import PcgConfig, SchurOperator, explicit_euler_step, recover_an
    spec = C.config_spec(0)
    op = SchurOperator(C.make_problem(0), pcg=PcgConfig(rel_tol=1e-8), strategy="cspe", max_cols=5)
    op.set_probe()
    a, t = np.zeros(op.grid.n_c), 0.0
    recover_an(op, a, t)
    for s in range(4):
        a, _ = explicit_euler_step((a, t), spec.dt, op, s + 1)
        t += spec.dt
        after_euler = op.probe_b()
        assert after_euler == op.probe_b(a)
        recover_an(op, a, t)
        cached = op.probe_b()
        assert cached == op.probe_b(a) == after_euler and cached > 0.0
    other = np.random.default_rng(5).standard_normal(op.grid.n_c)
    recover_an(op, a, t)
    assert op.probe_b() == op.probe_b(a)
    op._set_state(other, t)                        # the device state changed: recomputed
    assert op.probe_b() == op.probe_b(other) != op.probe_b(a)
    recover_an(op, a, t)
    cells = op.set_probe(op.probe_cells[:3])       # new cells: recomputed
    assert cells.size == 3 and op.probe_b(a) == op.probe_b(a)
    recover_an(op, a, t)
    assert op.probe_b() == op.probe_b(a)
    op.grid.close()


FIELD_CASES = {
    "cfg1_cspe": dict(index=1, strategy="cspe"),
    "cfg1_pod": dict(index=1, strategy="pod", n_pod=20),
    "cfg2": dict(index=2, strategy="pod", n_pod=30),
    "cfg3_m255": dict(index=3, strategy="cspe", member=255),
}


@pytest.mark.slow
@pytest.mark.parametrize("case", list(FIELD_CASES))
def test_config_fields_vs_oracle(gpu_ok, case):
    """The north-star bar at config scale: the A-field (a_c, a_n) of every
    step within 1e-8 relative L2 of the CPU oracle's run, every solve within
    +-1 iteration.  Fixtures (tests/golden/make_oracle_fields.py): configs[1]
    100 steps CSPE k = 5 and 60 steps POD-20 (rings full and evicting),
    configs[2] 25 steps (128^3, POD-30), configs[3] member 255 20 steps.  Per
    step the fixture holds ||A_ref|| and a CountSketch of A_ref
    (tests/fieldcheck.py: an unbiased estimate of ||A - A_ref||, 2 % relative
    spread); the last step holds the full field, where the exact error is
    checked as well and the estimate is checked against it."""
    from paper_1611_06721_b200 import configs as C
    from paper_1611_06721_b200 import PcgConfig, run_explicit
    from paper_1611_06721_b200 import ensemble as E
    from tests import fieldcheck as F
    c = FIELD_CASES[case]
    ref = np.load(Path(__file__).parent / "golden" / f"fields_{case}.npz")
    steps, dt = int(ref["steps"]), float(ref["dt"])
    if "member" in c:
        prob, _, _, dt_m = E.member_problem(c["member"])
        assert dt_m == dt
    else:
        prob = C.make_problem(c["index"])
        assert C.config_spec(c["index"]).dt == dt
    res = run_explicit(prob, t_end=steps * dt, dt=dt, strategy=c["strategy"], pcg=PcgConfig(rel_tol=1e-8),
                       max_cols=5, n_pod=c.get("n_pod", 10), eps_pod=1e-4,
                       output_period=dt * (1 - 1e-3), record_states=True)
    n_c, n_n = int(ref["n_c"]), int(ref["n_n"])
    assert res.a_c_history.shape == (steps, n_c) and res.a_n_history.shape == (steps, n_n)
    plan = F.sketch_plan(n_c + n_n)
    est = np.array([F.sketched_rel(F.field_of(res.a_c_history[i], res.a_n_history[i]), ref["sketch"][i + 1],
                                   ref["norm"][i + 1], plan) for i in range(steps)])
    assert est.max() <= REL_FIELD, (int(est.argmax()) + 1, float(est.max()))
    # exact checks at the last step
    assert rel(res.final_a_c, ref["a_c_final"]) <= REL_FIELD
    if "a_n_final" in ref:
        exact = F.exact_rel(F.field_of(res.final_a_c, res.final_a_n),
                            F.field_of(ref["a_c_final"], ref["a_n_final"]))
        assert exact <= REL_FIELD
        assert abs(est[-1] / exact - 1.0) <= 0.2, (est[-1], exact)
    it = res.step_iterations
    src = ref["iters_src"][1:].reshape(steps, 2)
    assert np.max(np.abs(it[:, 0] - src[:, 0])) <= 1 and np.max(np.abs(it[:, 2] - src[:, 1])) <= 1
    assert np.max(np.abs(it[:, 1] - ref["iters_prev"])) <= 1
    assert np.max(np.abs(it[:, 3] - ref["iters_cur"][1:])) <= 1


def test_cfl_estimate_matches_oracle_and_reference(gpu_ok, golden):
    """estimate_cfl (schur.py:327-376) on the device vs the oracle and the
    reference's own lambda (golden) at config 0."""
    from paper_1611_06721_b200 import configs as C
    from paper_1611_06721_b200 import PcgConfig, SchurOperator, estimate_cfl
    spec, m = oracle_model(0)
    op = SchurOperator(C.make_problem(0), pcg=PcgConfig(rel_tol=1e-8), strategy="cspe", max_cols=5)
    est = estimate_cfl(op, safety=0.9, seed=42)
    lam_ref, dt_ref, used_ref = golden["c0_cfl"]
    assert est.power_iters == int(used_ref)
    assert abs(est.lambda_max - lam_ref) <= 1e-9 * lam_ref
    assert abs(est.dt_max - dt_ref) <= 1e-9 * dt_ref
    # zero / wrong-shape start vectors reseed deterministically (schur.py:344-354)
    est0 = estimate_cfl(op, v0=np.zeros(m.n_c))
    assert est0.lambda_max == est.lambda_max
    with pytest.raises(ValueError):
        estimate_cfl(op, safety=1.5)
    # a saturated reference state lowers nu... and raises lambda
    ref = O.SchurOracle(m, O.sinusoid(50.0), "cspe", 1e-8, 5000, 5)
    a_ref = np.random.default_rng(1).standard_normal(m.n_c) * 1e-4
    lam_o, dt_o, used_o = ref.estimate_cfl(a_ref=a_ref)
    est_a = estimate_cfl(op, a_c_ref=a_ref)
    assert abs(est_a.lambda_max - lam_o) <= 1e-8 * lam_o


@pytest.mark.slow
def test_ensemble_member_first_steps(gpu_ok):
    """configs[3] member 1 (J, kappa factors, dt scaled with kappa): two
    device steps against the oracle on the same perturbed problem."""
    from paper_1611_06721_b200 import PcgConfig, run_explicit
    from paper_1611_06721_b200 import ensemble as E
    prob, jf, kf, dt = E.member_problem(1)
    spec, m = oracle_model(3, j_scale=jf, kappa_scale=kf)
    tr = O.run(m, O.sinusoid(50.0), dt, 2, strategy="cspe", rel_tol=1e-8, max_cols=5)
    res = run_explicit(prob, t_end=2 * dt, dt=dt, strategy="cspe", pcg=PcgConfig(rel_tol=1e-8),
                       output_period=dt * (1 - 1e-3), max_cols=5, record_states=True)
    for i in range(2):
        assert rel(res.a_c_history[i], tr.a_c[i + 1]) <= REL_FIELD


@pytest.mark.parametrize("variant", ["simple", "brick", "brick2", "brick-mixed", "resident", "resident2"])
def test_pcg_kernel_variants_agree(gpu_ok, variant, monkeypatch):
    """All fused-PCG kernels (thread-per-row, TMA brick, shared-memory
    resident, each with one or -- MQ_PCG_SYNC=2 -- two grid reductions per
    iteration; brick-mixed: the opt-in mixed i-chunking, MQ_BRICK_MIX=1)
    solve the same system like the oracle; they differ only in the
    dot-product summation order (and, single-reduction, beta from the
    extrapolated r.z)."""
    from paper_1611_06721_b200 import PcgConfig, Preconditioner, pcg_solve
    from paper_1611_06721_b200 import configs as C
    from paper_1611_06721_b200.device import DeviceGrid
    kernel, _, mode = variant.partition("-")
    monkeypatch.setenv("MQ_PCG_KERNEL", kernel.rstrip("2"))
    monkeypatch.setenv("MQ_PCG_SYNC", "2" if kernel.endswith("2") else "1")
    monkeypatch.setenv("MQ_BRICK_MIX", "1" if mode == "mixed" else "0")
    for index in (0, 1):
        spec, m = oracle_model(index)
        with DeviceGrid(C.make_problem(index)) as g:
            rng = np.random.default_rng(17)
            b = m.kn @ rng.standard_normal(m.n_n)
            x0 = rng.standard_normal(m.n_n) * 1e-3
            inv = O.jacobi_inverse(m.kn.diagonal())
            for start in (None, x0):
                x, rep = pcg_solve(g.kn_operator(), b, x0=start,
                                   config=PcgConfig(rel_tol=1e-8, preconditioner=Preconditioner.JACOBI))
                ref = O.pcg(m.kn_apply, b, x0=start, rel_tol=1e-8, inv_diag=inv)
                assert rep.converged and abs(rep.iterations - ref.iterations) <= 1
                assert rel(x, ref.x) <= 1e-8


@pytest.mark.parametrize("kernel,sync", [("resident", "1"), ("resident", "2"), ("brick", "1"), ("brick", "2")])
def test_resident_pcg_semantics(gpu_ok, kernel, sync, monkeypatch):
    """64^3 (shared-memory resident and TMA brick kernels, one or two
    reductions per iteration): krylov.py's budget exhaustion, exact start
    vector, zero rhs and application counts, against the oracle.  The
    single-reduction kernels read the stopping test one barrier late; the
    counts must not see it."""
    from paper_1611_06721_b200 import PcgConfig, Preconditioner, pcg_solve
    from paper_1611_06721_b200 import configs as C
    from paper_1611_06721_b200.device import DeviceGrid
    monkeypatch.setenv("MQ_PCG_KERNEL", kernel)
    monkeypatch.setenv("MQ_PCG_SYNC", sync)
    spec, m = oracle_model(1)
    inv = O.jacobi_inverse(m.kn.diagonal())
    with DeviceGrid(C.make_problem(1)) as g:
        name, _ = g.pcg_kernel()
        want = {("resident", "1"): "pcg_resident1_kernel", ("resident", "2"): "pcg_resident_kernel",
                ("brick", "1"): "pcg_tma1_kernel", ("brick", "2"): "pcg_tma_kernel"}[(kernel, sync)]
        assert name.startswith(want), name
        op = g.kn_operator()
        jac = Preconditioner.JACOBI
        for budget in (1, 2, 3):
            x, rep = pcg_solve(op, m.pattern, config=PcgConfig(rel_tol=1e-14, max_iter=budget, preconditioner=jac))
            ref = O.pcg(m.kn_apply, m.pattern, rel_tol=1e-14, max_iter=budget, inv_diag=inv)
            assert not rep.converged and rep.iterations == budget and rep.applications == ref.applies
            assert rel(x, ref.x) <= 1e-12
            assert abs(rep.final_rel_residual - ref.rel) <= 1e-10 * ref.rel
        x, rep = pcg_solve(op, np.zeros(m.n_n), config=PcgConfig(rel_tol=1e-8, preconditioner=jac))
        assert rep.iterations == 0 and rep.converged and rep.applications == 0
        assert np.array_equal(x, np.zeros(m.n_n))
        ref = O.pcg(m.kn_apply, m.pattern, rel_tol=1e-8, inv_diag=inv)
        x, rep = pcg_solve(op, m.pattern, config=PcgConfig(rel_tol=1e-8, preconditioner=jac))
        assert rep.converged and abs(rep.iterations - ref.iterations) <= 1
        assert rep.applications == rep.iterations and rel(x, ref.x) <= 1e-8
        # warm start from the converged solution: 0 iterations, x unchanged
        b = m.kn @ x
        x2, rep2 = pcg_solve(op, b, x0=x, config=PcgConfig(rel_tol=1e-8, preconditioner=jac))
        assert rep2.iterations == 0 and rep2.applications == 1 and np.array_equal(x2, x)


@pytest.mark.parametrize("kernel,sync", [("resident", "1"), ("resident", "2"), ("brick", "1"), ("brick", "2")])
def test_pcg_barrier_stress(gpu_ok, kernel, sync, monkeypatch):
    """Race check of the persistent kernels' halo exchange: with MQ_PCG_STRESS a
    pseudo-random subset of CTAs sleeps 20 us after every grid barrier, so
    their neighbours run ahead into the next iteration's publication.  The
    solve depends on no timing: x and the iteration count are bit-identical
    to the unstressed solve (the single-reduction kernel once overwrote the
    Ap a delayed neighbour still had to load)."""
    from paper_1611_06721_b200 import PcgConfig, Preconditioner, pcg_solve
    from paper_1611_06721_b200 import configs as C
    from paper_1611_06721_b200.device import DeviceGrid
    monkeypatch.setenv("MQ_PCG_KERNEL", kernel)
    monkeypatch.setenv("MQ_PCG_SYNC", sync)
    prob = C.make_problem(1)
    with DeviceGrid(prob) as g:
        assert g.pcg_kernel()[0].startswith({"resident": "pcg_resident", "brick": "pcg_tma"}[kernel])
        op = g.kn_operator()
        rng = np.random.default_rng(11)
        b = g.kn_apply(rng.standard_normal(g.n_n))
        x0 = rng.standard_normal(g.n_n) * 1e-3
        cfg = PcgConfig(rel_tol=1e-8, preconditioner=Preconditioner.JACOBI)
        for start in (None, x0):
            monkeypatch.delenv("MQ_PCG_STRESS", raising=False)
            x, rep = pcg_solve(op, b, x0=start, config=cfg)
            monkeypatch.setenv("MQ_PCG_STRESS", "20000")
            xs, reps = pcg_solve(op, b, x0=start, config=cfg)
            assert rep.converged and reps.iterations == rep.iterations
            assert np.array_equal(xs, x)


@pytest.mark.parametrize("shape,li", [((33, 64, 64), 3), ((26, 64, 64), 2), ((48, 64, 48), 4),
                                      ((20, 128, 128), 5)])
@pytest.mark.parametrize("sync", ["1", "2"])
def test_resident_pcg_other_brick_depths(gpu_ok, shape, li, sync, monkeypatch):
    """Non-cubic grids whose resident bricks hold 2, 3, 4 or 5 i-planes (the
    kernel templates LI; 5 planes only fit the two-barrier kernel) and tiles
    cut by the grid edge: PCG against the oracle, cold and warm start."""
    from paper_1611_06721_b200 import PcgConfig, Preconditioner, pcg_solve
    from paper_1611_06721_b200.device import DeviceGrid, Problem
    monkeypatch.setenv("MQ_PCG_KERNEL", "resident")
    monkeypatch.setenv("MQ_PCG_SYNC", sync)
    mat = np.zeros(shape, np.int8)
    nx, ny, nz = shape
    mat[nx // 3:nx // 3 + 6, ny // 3:ny // 3 + 9, nz // 4:nz // 4 + 7] = 1
    h = 1.0 / max(shape)
    m = O.assemble(mat, h, O.Conductor(5e6, 3.8, 2.17, 396.2), [])
    inv = O.jacobi_inverse(m.kn.diagonal())
    rng = np.random.default_rng(sum(shape))
    b = m.kn @ rng.standard_normal(m.n_n)
    x0 = rng.standard_normal(m.n_n) * 1e-3
    with DeviceGrid(Problem(material=mat, h=h, kappa=5e6, brauer=(3.8, 2.17, 396.2),
                            pattern=np.zeros(m.n_n))) as g:
        name, _ = g.pcg_kernel()
        one = sync == "1" and li <= 4
        assert name == (f"pcg_resident1_kernel<{li}>" if one else f"pcg_resident_kernel<{li}>"), name
        for start in (None, x0):
            x, rep = pcg_solve(g.kn_operator(), b, x0=start,
                               config=PcgConfig(rel_tol=1e-8, preconditioner=Preconditioner.JACOBI))
            ref = O.pcg(m.kn_apply, b, x0=start, rel_tol=1e-8, inv_diag=inv)
            assert rep.converged and abs(rep.iterations - ref.iterations) <= 1
            assert rep.applications == ref.applies + (rep.iterations - ref.iterations)
            assert rel(x, ref.x) <= 1e-8


@pytest.mark.parametrize("sync", ["1", "2"])
@pytest.mark.parametrize("shape", [(150, 40, 40), (97, 24, 70)])
def test_tma_pcg_long_bricks(gpu_ok, shape, sync, monkeypatch):
    """TMA brick kernels on bricks longer than the shared-memory mask cache
    (MQ_BRICK_CHUNKS=1: one brick per tile column, 150 / 97 planes; the
    configs[4] case): the one-barrier kernel -- the default at every brick
    length -- takes the mask words from global memory there, odd plane counts
    end the two-plane unrolled march on a single step.  PCG against the oracle,
    cold and warm start, budget exhaustion."""
    from paper_1611_06721_b200 import PcgConfig, Preconditioner, pcg_solve
    from paper_1611_06721_b200.device import DeviceGrid, Problem
    monkeypatch.setenv("MQ_PCG_KERNEL", "brick")
    monkeypatch.setenv("MQ_PCG_SYNC", sync)
    monkeypatch.setenv("MQ_BRICK_CHUNKS", "1")
    mat = np.zeros(shape, np.int8)
    nx, ny, nz = shape
    mat[nx // 3:nx // 3 + 11, ny // 3:ny // 3 + 9, nz // 4:nz // 4 + 7] = 1
    h = 1.0 / max(shape)
    m = O.assemble(mat, h, O.Conductor(5e6, 3.8, 2.17, 396.2), [])
    inv = O.jacobi_inverse(m.kn.diagonal())
    rng = np.random.default_rng(sum(shape))
    b = m.kn @ rng.standard_normal(m.n_n)
    x0 = rng.standard_normal(m.n_n) * 1e-3
    jac = Preconditioner.JACOBI
    with DeviceGrid(Problem(material=mat, h=h, kappa=5e6, brauer=(3.8, 2.17, 396.2),
                            pattern=np.zeros(m.n_n))) as g:
        name, _ = g.pcg_kernel()
        assert name == ("pcg_tma1_kernel" if sync == "1" else "pcg_tma_kernel"), name
        for start in (None, x0):
            x, rep = pcg_solve(g.kn_operator(), b, x0=start, config=PcgConfig(rel_tol=1e-8, preconditioner=jac))
            ref = O.pcg(m.kn_apply, b, x0=start, rel_tol=1e-8, inv_diag=inv)
            assert rep.converged and abs(rep.iterations - ref.iterations) <= 1
            assert rep.applications == ref.applies + (rep.iterations - ref.iterations)
            assert rel(x, ref.x) <= 1e-8
        for budget in (1, 2, 3, 4):
            x, rep = pcg_solve(g.kn_operator(), b, config=PcgConfig(rel_tol=1e-14, max_iter=budget, preconditioner=jac))
            ref = O.pcg(m.kn_apply, b, rel_tol=1e-14, max_iter=budget, inv_diag=inv)
            assert not rep.converged and rep.iterations == budget and rep.applications == ref.applies
            assert rel(x, ref.x) <= 1e-12


@pytest.mark.parametrize("world", [1, 2, 3])
@pytest.mark.parametrize("x0_given", [False, True])
def test_slab_pcg_loopback_on_one_gpu(gpu_ok, world, x0_given):
    """configs[4] i-slab decomposition on one GPU: `world` slab contexts, halo
    exchange by device copies, fixed-order partial sums (LoopbackComm), the
    same host loop as the NCCL path.  Partition union bit-exact; solution vs
    the single-domain oracle."""
    from paper_1611_06721_b200 import configs as C
    from paper_1611_06721_b200.slab import LoopbackComm, SlabGrid, slab_pcg_solve
    spec, m = oracle_model(0)
    prob = C.make_problem(0)
    slabs = [SlabGrid(prob, r, world) for r in range(world)]
    parts = [s.partition() for s in slabs]
    allp = np.concatenate(parts)
    assert allp.size == m.n_n and np.array_equal(np.sort(allp), m.noncond_global)
    idx = [np.searchsorted(m.noncond_global, p) for p in parts]
    rng = np.random.default_rng(9)
    b = m.kn @ rng.standard_normal(m.n_n)
    x0 = rng.standard_normal(m.n_n) * 1e-3
    for s, ix in zip(slabs, idx):
        s.upload(b[ix], s.b)
        s.upload(x0[ix] if x0_given else np.zeros(ix.size), s.x)
    it, relres, conv, app = slab_pcg_solve(slabs, LoopbackComm(), x0_given=x0_given, rel_tol=1e-8)
    ref = O.pcg(m.kn_apply, b, x0=x0 if x0_given else None, rel_tol=1e-8,
                inv_diag=O.jacobi_inverse(m.kn.diagonal()))
    x = np.zeros(m.n_n)
    for s, ix in zip(slabs, idx):
        x[ix] = s.download(s.x)
    assert conv and abs(it - ref.iterations) <= 1 and app == ref.applies - (ref.iterations - it)
    assert rel(x, ref.x) <= 1e-8
    for s in slabs:
        s.close()


@pytest.mark.parametrize("world", [1, 2, 3, 4])
@pytest.mark.parametrize("x0_given", [False, True])
@pytest.mark.parametrize("sync", ["1", "2"])
def test_fused_slab_pcg_on_one_gpu(gpu_ok, world, x0_given, sync, monkeypatch):
    """The fused per-rank slab kernels (ghost stores into the neighbour slab,
    rank all-reduce through device mailboxes; one all-reduce per iteration --
    pcg_tma1_slab_kernel -- or, MQ_PCG_SYNC=2, two), their ranks emulated as
    the CTA groups of one cooperative launch: solution vs the single-domain
    oracle, iterations within +-1, application counts; repeated solves reuse
    the mailboxes (epochs)."""
    from paper_1611_06721_b200 import configs as C
    from paper_1611_06721_b200.slab import SlabGrid, fused_slab_pcg_solve_local
    monkeypatch.setenv("MQ_PCG_SYNC", sync)
    spec, m = oracle_model(0)
    prob = C.make_problem(0)
    slabs = [SlabGrid(prob, r, world) for r in range(world)]
    idx = [np.searchsorted(m.noncond_global, s.partition()) for s in slabs]
    rng = np.random.default_rng(11)
    inv = O.jacobi_inverse(m.kn.diagonal())
    for rep in range(3):
        b = m.kn @ rng.standard_normal(m.n_n)
        x0 = rng.standard_normal(m.n_n) * 1e-3
        for s, ix in zip(slabs, idx):
            s.upload(b[ix], s.b)
            s.upload(x0[ix] if x0_given else np.zeros(ix.size), s.x)
        it, relres, conv, app = fused_slab_pcg_solve_local(slabs, x0_given=x0_given, rel_tol=1e-8)
        ref = O.pcg(m.kn_apply, b, x0=x0 if x0_given else None, rel_tol=1e-8, inv_diag=inv)
        x = np.zeros(m.n_n)
        for s, ix in zip(slabs, idx):
            x[ix] = s.download(s.x)
        assert conv and abs(it - ref.iterations) <= 1, (it, ref.iterations)
        assert app == ref.applies - (ref.iterations - it)
        assert rel(x, ref.x) <= 1e-8
    for s in slabs:
        s.close()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("sync", ["1", "2"])
def test_fused_slab_barrier_stress(gpu_ok, world, sync, monkeypatch):
    """The fused slab kernel with some CTAs of every rank group delayed after
    each rank all-reduce (MQ_PCG_STRESS): ghost stores into the neighbours'
    slabs and the mailbox protocol depend on no timing, so x and the
    iteration count are bit-identical to the unstressed solve."""
    from paper_1611_06721_b200 import configs as C
    from paper_1611_06721_b200.slab import SlabGrid, fused_slab_pcg_solve_local
    monkeypatch.setenv("MQ_PCG_SYNC", sync)
    spec, m = oracle_model(0)
    prob = C.make_problem(0)
    slabs = [SlabGrid(prob, r, world) for r in range(world)]
    idx = [np.searchsorted(m.noncond_global, s.partition()) for s in slabs]
    rng = np.random.default_rng(19)
    b = m.kn @ rng.standard_normal(m.n_n)
    out = []
    for stress in (None, "20000"):
        if stress:
            monkeypatch.setenv("MQ_PCG_STRESS", stress)
        else:
            monkeypatch.delenv("MQ_PCG_STRESS", raising=False)
        for s, ix in zip(slabs, idx):
            s.upload(b[ix], s.b)
            s.upload(np.zeros(ix.size), s.x)
        it, relres, conv, app = fused_slab_pcg_solve_local(slabs, x0_given=False, rel_tol=1e-8)
        x = np.zeros(m.n_n)
        for s, ix in zip(slabs, idx):
            x[ix] = s.download(s.x)
        assert conv
        out.append((it, x))
    assert out[0][0] == out[1][0] and np.array_equal(out[0][1], out[1][1])
    for s in slabs:
        s.close()


@pytest.mark.parametrize("sync", ["1", "2"])
def test_fused_slab_peer_path_single_rank(gpu_ok, sync, monkeypatch):
    """The one-rank-per-process entry points (IPC export/import, the kernel
    launched as a single CTA group) at one rank: same answer as the oracle.
    (More ranks need more GPUs; the protocol is the one the emulated
    multi-group launches above exercise.)"""
    from paper_1611_06721_b200 import configs as C
    from paper_1611_06721_b200.slab import SlabGrid, fused_peer_setup, fused_peer_solve
    monkeypatch.setenv("MQ_PCG_SYNC", sync)
    spec, m = oracle_model(0)
    s = SlabGrid(C.make_problem(0), 0, 1)
    fused_peer_setup(s)
    rng = np.random.default_rng(13)
    inv = O.jacobi_inverse(m.kn.diagonal())
    for x0_given in (False, True, False):
        b = m.kn @ rng.standard_normal(m.n_n)
        x0 = rng.standard_normal(m.n_n) * 1e-3
        s.upload(b, s.b)
        s.upload(x0 if x0_given else np.zeros(m.n_n), s.x)
        it, relres, conv, app = fused_peer_solve(s, x0_given=x0_given, rel_tol=1e-8)
        ref = O.pcg(m.kn_apply, b, x0=x0 if x0_given else None, rel_tol=1e-8, inv_diag=inv)
        assert conv and abs(it - ref.iterations) <= 1
        assert rel(s.download(s.x), ref.x) <= 1e-8
    s.close()


@pytest.mark.slow
def test_fused_slab_pcg_config1_grid(gpu_ok):
    """64^3 (configs[1] grid) split over 4 emulated ranks: the cold source
    solve against the single-context device solve."""
    from paper_1611_06721_b200 import PcgConfig, configs as C, pcg_solve
    from paper_1611_06721_b200.device import DeviceGrid
    from paper_1611_06721_b200.slab import SlabGrid, fused_slab_pcg_solve_local
    prob = C.make_problem(1)
    with DeviceGrid(prob) as g:
        nc_all = g.partition()[0]
        x_ref, rep_ref = pcg_solve(g.kn_operator(), prob.pattern, config=PcgConfig(rel_tol=1e-8))
    slabs = [SlabGrid(prob, r, 4) for r in range(4)]
    idx = [np.searchsorted(nc_all, s.partition()) for s in slabs]
    for s, ix in zip(slabs, idx):
        s.upload(prob.pattern[ix], s.b)
    it, relres, conv, app = fused_slab_pcg_solve_local(slabs, x0_given=False, rel_tol=1e-8)
    x = np.zeros(nc_all.size)
    for s, ix in zip(slabs, idx):
        x[ix] = s.download(s.x)
    assert conv and abs(it - rep_ref.iterations) <= 1
    assert rel(x, x_ref) <= 1e-8
    for s in slabs:
        s.close()


@pytest.mark.gpu
def test_concurrent_members_match_sequential(gpu_ok):
    """configs[3] members stepped side by side on SM slices (ensemble.run_members)
    follow the same trajectories as one member on the whole GPU: fields within
    the north-star bar, iteration counts within +-1 per solve (the slice
    changes only the dot products' reduction order)."""
    from paper_1611_06721_b200 import ensemble as E
    steps = 6
    conc = E.run_members([0, 1, 2], steps, concurrency=3)
    for r in conc:
        ref = E.run_member(r.member, steps)
        assert abs(r.final_norm_a_c - ref.final_norm_a_c) <= REL_FIELD * ref.final_norm_a_c
        for fam, v in ref.iterations.items():
            assert abs(r.iterations[fam] - v) <= 2 * steps + 1, (fam, r.iterations, ref.iterations)


def _guard(lib, ctx):
    import ctypes
    bad, nv, chk = ctypes.c_int64(), ctypes.c_int32(), ctypes.c_int32()
    from paper_1611_06721_b200._lib import check
    check(lib.mq_guard_check(ctx, ctypes.byref(bad), ctypes.byref(nv), ctypes.byref(chk)))
    return bad.value, nv.value, chk.value


@pytest.mark.parametrize("index,strategy,steps", [(0, "cspe", 20), (0, "pod", 20), (0, "previous", 10),
                                                  (1, "cspe", 4), (1, "pod", 4), (2, "pod", 2)])
def test_guard_entries_stay_zero(gpu_ok, index, strategy, steps):
    """Memory-safety evidence in place of compute-sanitizer (closed on this
    pool): after a run, every off-partition entry of every device vector of
    the context (PCG scratch, CSPE / POD caches, work vectors) is still 0 —
    the stencils read them as boundary values, so a stray or out-of-range
    write into the padded layout would show here (and in the results)."""
    from paper_1611_06721_b200 import configs as C
    from paper_1611_06721_b200 import PcgConfig, SchurOperator, run_explicit
    spec = C.config_spec(index)
    op = SchurOperator(C.make_problem(index), pcg=PcgConfig(rel_tol=1e-8), strategy=strategy, max_cols=5,
                       n_pod=20 if index < 2 else 30)
    run_explicit(op.problem, t_end=steps * spec.dt, dt=spec.dt, output_period=spec.dt * (1 - 1e-3), op=op)
    bad, nv, chk = _guard(op.lib, op.grid.ctx)
    assert chk > 10 and bad == 0, (bad, nv, chk)
    op.grid.close()


def test_guard_entries_stay_zero_on_slabs(gpu_ok):
    """The same on the slabs of the sharded step (ghost planes excepted)."""
    from paper_1611_06721_b200 import configs as C
    from paper_1611_06721_b200.slabstep import SlabStepper, run_explicit_sharded
    spec = C.config_spec(0)
    st = SlabStepper(C.make_problem(0), 3, strategy="cspe", max_cols=5)
    try:
        run_explicit_sharded(st.problem, 8, spec.dt, world=3, stepper=st)
        for s in st.slabs:
            bad, nv, chk = _guard(s.lib, s.ctx)
            assert chk >= 5 and bad == 0, (bad, nv, chk)
    finally:
        st.close()
