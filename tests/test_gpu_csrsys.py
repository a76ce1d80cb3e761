"""Models given as matrices on the GPU: a CSR block
resident on the device (mq_csr_op_*) for PCG solves and SpMVs, and the
frozen-linear system of a reference manifest stepped with every K_n solve on
the device, against the CPU oracle (oracle.mq_oracle.SchurOracle over the
same CSR blocks).  Bars as in test_gpu_parity: field 1e-8 relative, PCG
iterations +-1."""
from pathlib import Path

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import mq_oracle as O
from tests.conftest import oracle_model

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"
REL_FIELD = 1e-8


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / (nb if nb > 0 else 1.0)


def fixture_system():
    from paper_1611_06721_b200.csrsys import load_manifest
    return load_manifest(GOLD / "manifest_c6")


def config0_system():
    """configs[0] (16^3, linear iron, sinusoidal coil) as a matrix system:
    the oracle's K_n, K_cn, M_c and K_c (linear: one matrix), the BASELINE
    waveform as the manifest's sinusoid kind."""
    from paper_1611_06721_b200.csrsys import CsrSystem, sinusoid_waveform
    spec, m = oracle_model(0)
    eye = np.eye(m.n_c)
    kc = sp.csr_matrix(np.column_stack([m.kc_apply(np.zeros(m.n_c), eye[:, j]) for j in range(m.n_c)]))
    kc.eliminate_zeros()
    return spec, m, CsrSystem(mc=sp.diags(m.mc_diag).tocsr(), kc=kc, kcn=m.kcn.tocsr(), kn=m.kn.tocsr(),
                              pattern=m.pattern.copy(), waveform=sinusoid_waveform(50.0))


def test_csr_operator_spmv_and_pcg(gpu_ok):
    from paper_1611_06721_b200 import PcgConfig, Preconditioner, pcg_solve
    from paper_1611_06721_b200.csrsys import CsrOperator
    for s in (fixture_system(), config0_system()[2]):
        kn = s.kn
        with CsrOperator(kn) as op:
            rng = np.random.default_rng(kn.shape[0])
            x = rng.standard_normal(op.n)
            assert np.array_equal(op(x), kn @ x)          # CSR row order, like scipy's csr_matvec
            b = kn @ rng.standard_normal(op.n)
            inv = O.jacobi_inverse(kn.diagonal())
            for start in (None, rng.standard_normal(op.n) * 1e-3):
                xs, rep = pcg_solve(op, b, x0=start,
                                    config=PcgConfig(rel_tol=1e-8, preconditioner=Preconditioner.JACOBI))
                ref = O.pcg(lambda v: kn @ v, b, x0=start, rel_tol=1e-8, inv_diag=inv)
                assert rep.converged and abs(rep.iterations - ref.iterations) <= 1
                assert rep.applications == ref.applies + (rep.iterations - ref.iterations)
                assert rel(xs, ref.x) <= 1e-8
            # budget exhaustion and a non-rectangular block
            xs, rep = op.solve(b, config=PcgConfig(rel_tol=1e-14, max_iter=2))
            ref = O.pcg(lambda v: kn @ v, b, rel_tol=1e-14, max_iter=2, inv_diag=inv)
            assert not rep.converged and rep.iterations == 2 and rel(xs, ref.x) <= 1e-12
        with CsrOperator(s.kcn.T, jacobi=False) as opt:
            y = np.random.default_rng(3).standard_normal(s.n_c)
            assert opt.shape == (s.n_n, s.n_c)
            assert rel(opt(y), s.kcn.T @ y) <= 1e-15


@pytest.mark.parametrize("which", ["fixture", "config0"])
@pytest.mark.parametrize("strategy", ["previous", "zero"])
def test_csr_system_steps_vs_oracle(gpu_ok, which, strategy):
    """run_explicit over the CSR system: every step's a_c and the recovered
    a_n within the field bar of the oracle's run, iteration counts +-1."""
    from paper_1611_06721_b200 import PcgConfig
    from paper_1611_06721_b200.csrsys import run_explicit
    if which == "fixture":
        s = fixture_system()
        dt, n = 2e-4, 8
    else:
        spec, _, s = config0_system()
        dt, n = spec.dt, 5
    res = run_explicit(s, t_end=n * dt, dt=dt, strategy=strategy, pcg=PcgConfig(rel_tol=1e-8),
                       output_period=dt * (1 - 1e-3), record_states=True)
    model = O.CsrModel(kn=s.kn, kcn=s.kcn, kc=s.kc, mc_diag=s.mc.diagonal(), pattern=s.pattern)
    tr = O.run(model, s.waveform, dt, n, strategy=strategy, rel_tol=1e-8)
    assert len(res.a_c_history) == n
    for i in range(n):
        assert rel(res.a_c_history[i], tr.a_c[i + 1]) <= REL_FIELD, i
    assert rel(res.final_a_n, tr.a_n[-1]) <= 5e-8
    assert np.linalg.norm(res.final_a_c) > 0
    for a, b in ((res.iters_src, tr.iters[O.FAM_SOURCE][1::2]), (res.iters_cpl_prev, tr.iters[O.FAM_PREV]),
                 (res.iters_cpl_cur, tr.iters[O.FAM_CUR][1:])):
        assert np.max(np.abs(np.asarray(a) - np.asarray(b))) <= 1


def test_csr_strategy_object(gpu_ok):
    """A StartVectorStrategy object (protocol startvec.py:315-342) drives the
    start vectors: the oracle's CSPE cache behind the protocol names."""
    from paper_1611_06721_b200 import PcgConfig
    from paper_1611_06721_b200.csrsys import CsrSchurOperator, explicit_euler_step, recover_an
    s = fixture_system()
    cspe = O.make_strategy("cspe", s.n_n, lambda v: s.kn @ v, max_cols=5, drop_tol=1e-8)

    class Protocol:
        kind = "cspe"

        def start_vector(self, family, rhs):
            return cspe.start(family.value, rhs)

        def observe(self, family, solution):
            cspe.observe(family.value, solution)

    op = CsrSchurOperator(s, pcg=PcgConfig(rel_tol=1e-8), strategy=Protocol())
    a, t, dt = np.zeros(s.n_c), 0.0, 2e-4
    recover_an(op, a, t)
    for k in range(6):
        a, (r1, r2) = explicit_euler_step((a, t), dt, op, k + 1)
        t += dt
        recover_an(op, a, t)
    # the source family's span holds the pattern: its solves start exact
    from paper_1611_06721_b200 import RhsFamily
    assert op.solve_iterations[RhsFamily.SOURCE_CURRENT][-1] <= 1
    assert cspe.basis_size() > 0
    op.close()


def _with_builtin(tmp_path, **over):
    import json
    import shutil
    d = tmp_path / "m"
    shutil.copytree(GOLD / "manifest_c6", d)
    mf = json.loads((d / "manifest.json").read_text())
    mf["builtin"] = {"cells": 6, "h": 5e-3, "kappa": 5e6, "brauer": [49.4, 1.46, 520.6], "amps": 50000.0,
                     "tau": 0.5, "linear": False, "probe_cells": None, **over}
    (d / "manifest.json").write_text(json.dumps(mf))
    return d


def test_builtin_manifest_blocks_checked_on_device(gpu_ok, tmp_path):
    """bench.py:283-306: a manifest's builtin section rebuilds the FIT model;
    stored blocks that disagree are refused, and the nonlinear model is not
    stepped as frozen-linear (its stencil-path Problem is system.builtin)."""
    import scipy.io
    from paper_1611_06721_b200.csrsys import ConfigError, CsrSchurOperator, load_manifest, verify_builtin
    s = load_manifest(_with_builtin(tmp_path / "a"))
    verify_builtin(s)                                    # the stored blocks are builtin_model(6)'s
    with pytest.raises(ConfigError, match="nonlinear"):
        CsrSchurOperator(s)
    op = CsrSchurOperator(load_manifest(_with_builtin(tmp_path / "b", linear=True)))  # K_c(0) is the linear K_c
    op.close()
    d = _with_builtin(tmp_path / "c", linear=True)
    kn = scipy.io.mmread(str(d / "k_n.mtx")).tocsr()
    kn.data[0] *= 1.0 + 1e-12
    scipy.io.mmwrite(str(d / "k_n.mtx"), kn, symmetry="general")
    with pytest.raises(ConfigError, match="'k_n'"):
        CsrSchurOperator(load_manifest(d))


def test_consistent_mass_solve(gpu_ok):
    """A non-diagonal M_c takes the reference's Jacobi-PCG mass solve
    (schur.py:210-218, 280-287) instead of 1/diag."""
    from paper_1611_06721_b200 import PcgConfig
    from paper_1611_06721_b200.csrsys import CsrSchurOperator, CsrSystem, explicit_euler_step
    base = fixture_system()
    d = base.mc.diagonal()
    off = 0.1 * np.minimum(d[:-1], d[1:])
    mc = sp.diags([off, d, off], [-1, 0, 1]).tocsr()
    s = CsrSystem(mc=mc, kc=base.kc, kcn=base.kcn, kn=base.kn, pattern=base.pattern, waveform=base.waveform)
    op = CsrSchurOperator(s, pcg=PcgConfig(rel_tol=1e-10), strategy="zero")
    try:
        assert op.minv_diag is None
        rng = np.random.default_rng(2)
        a = rng.standard_normal(s.n_c) * 1e-3
        inv_kn = O.jacobi_inverse(s.kn.diagonal())
        dt = 2e-4
        y_src = O.pcg(lambda v: s.kn @ v, s.pattern * s.waveform(dt), rel_tol=1e-10, inv_diag=inv_kn).x
        y_cpl = O.pcg(lambda v: s.kn @ v, s.kcn.T @ a, rel_tol=1e-10, inv_diag=inv_kn).x
        rate = s.kcn @ (y_cpl - y_src) - s.kc @ a
        ref = a + dt * O.pcg(lambda v: mc @ v, rate, rel_tol=1e-10, inv_diag=O.jacobi_inverse(d)).x
        got, _ = explicit_euler_step((a, 0.0), dt, op)
        assert rel(got, ref) <= 1e-9
        # 1/diag would be visibly different
        assert rel(a + dt * rate / d, ref) > 1e-6
    finally:
        op.close()
