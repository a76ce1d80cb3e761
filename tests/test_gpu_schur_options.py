"""The reference's SchurOperator options on the device twin, against the
reference's own runs (tests/golden/make_golden_options.py, config 0, CSPE
k = 5, 20 steps, an output row per step):

* ``cache_source_solve=True`` (schur.py:266-278): one pattern solve, rescaled;
* ``projection_target="composed-coupling"`` (schur.py:244-250);
* ``strategy=<StartVectorStrategy object>`` (schur.py:198-199): a host-side
  strategy (here the oracle's CSPE cache behind the reference's protocol)
  with every PCG solve and product on the device;
* ``apply`` / ``apply_detached`` (schur.py:289-313) and
  ``aggregates["solver_seconds"]`` (schur.py:592).
"""

from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

from oracle import mq_oracle as O
from tests.conftest import oracle_model

pytestmark = pytest.mark.gpu

GOLD = Path(__file__).parent / "golden" / "reference_options.npz"


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


class OracleCspeAdapter:
    """The reference's StartVectorStrategy protocol (startvec.py:315-342) over
    the oracle's CSPE cache (test infrastructure standing in for a user's
    strategy object)."""

    kind = "cspe"

    def __init__(self, m, max_cols=5, drop_tol=1e-8):
        self.s = O.CspeStrategyOracle(m.n_n, m.kn_apply, max_cols=max_cols, drop_tol=drop_tol)

    def start_vector(self, family, rhs):
        return self.s.start(family, np.asarray(rhs))

    def observe(self, family, solution):
        self.s.observe(family, np.asarray(solution))

    def basis_size(self, family=None):
        return self.s.basis_size()

    @property
    def maintenance_applies(self):
        return self.s.maintenance

    def diagnostics(self):
        return self.s.diagnostics()


def _compare(res, ref, key):
    n = int(ref["nsteps"])
    assert res.n_rows == n + 1
    assert np.array_equal(res.times, ref[f"{key}_times"])
    assert rel(res.final_a_c, ref[f"{key}_final_a_c"]) <= 1e-8
    assert rel(np.concatenate([res.final_a_c, res.final_a_n]),
               np.concatenate([ref[f"{key}_final_a_c"], ref[f"{key}_final_a_n"]])) <= 1e-8
    assert rel(res.probe_b, ref[f"{key}_probe_b"]) <= 1e-8
    for col in ("iters_src", "iters_cpl_prev", "iters_cpl_cur"):
        assert np.max(np.abs(getattr(res, col) - ref[f"{key}_{col}"])) <= 1, col
    assert np.array_equal(res.basis_cols, ref[f"{key}_basis_cols"])
    assert res.aggregates["solver_seconds"] > 0.0


@pytest.mark.parametrize("key", ["cache_src", "composed", "instance"])
def test_schur_options_match_reference(gpu_ok, key):
    from paper_1611_06721_b200 import configs as C
    from paper_1611_06721_b200 import PcgConfig, run_explicit
    ref = np.load(GOLD)
    spec, m = oracle_model(0)
    dt, n = float(ref["dt"]), int(ref["nsteps"])
    kw = {"cache_src": dict(strategy="cspe", cache_source_solve=True),
          "composed": dict(strategy="cspe", projection_target="composed-coupling"),
          "instance": dict(strategy=OracleCspeAdapter(m))}[key]
    res = run_explicit(C.make_problem(0), t_end=n * dt, dt=dt, pcg=PcgConfig(rel_tol=1e-8, max_iter=5000),
                       output_period=dt * (1 - 1e-3), probe="device", max_cols=5, **kw)
    _compare(res, ref, key)
    if key == "cache_src":
        # one pattern solve, then zero-iteration rescalings (schur.py:270-276)
        assert res.aggregates["solves"]["source"] == 1


def test_apply_and_apply_detached(gpu_ok):
    from paper_1611_06721_b200 import configs as C
    from paper_1611_06721_b200 import PcgConfig, SchurOperator
    from paper_1611_06721_b200.startvec import RhsFamily
    spec, m = oracle_model(0)
    op = SchurOperator(C.make_problem(0), pcg=PcgConfig(rel_tol=1e-10), strategy="cspe", max_cols=5)
    x = np.random.default_rng(11).standard_normal(m.n_c)
    ref_y = O.pcg(m.kn_apply, m.kcn.T @ x, rel_tol=1e-10, inv_diag=O.jacobi_inverse(m.kn.diagonal())).x
    ref = m.kc_apply(np.zeros(m.n_c), x) - m.kcn @ ref_y
    ks, y = op.apply_detached(x, np.zeros(m.n_c))
    assert rel(y, ref_y) <= 1e-8 and rel(ks, ref) <= 1e-8
    assert op.solve_count(RhsFamily.COUPLING_FROM_PREVIOUS_STATE) == 0   # no family history
    ks2 = op.apply(x, np.zeros(m.n_c))
    assert rel(ks2, ref) <= 1e-8
    assert op.solve_count(RhsFamily.COUPLING_FROM_PREVIOUS_STATE) == 1
    op.grid.close()
