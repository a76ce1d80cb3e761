"""Member-batched PCG (configs[3]): nb right-hand sides of the
same K_n in one launch, interleaved [entry][member], per-member scalars and
stopping; every member against its own single-member device solve (itself
pinned to the oracle): iterations within +-1, solutions within 1e-8."""

from __future__ import annotations

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("nb", [1, 2, 4, 8])
def test_batched_members_match_single_solves(gpu_ok, nb):
    from paper_1611_06721_b200 import _lib
    from paper_1611_06721_b200 import configs as C
    from paper_1611_06721_b200._lib import check, dptr
    from paper_1611_06721_b200.device import DeviceGrid
    with DeviceGrid(C.make_problem(0)) as g:
        rng = np.random.default_rng(nb)
        # members with different right-hand sides and scales (ensemble members
        # differ in J and kappa): consistent rhs K_n v
        b = np.stack([g.kn_apply(rng.standard_normal(g.n_n)) * (1.0 + 0.2 * m) for m in range(nb)])
        x0 = np.stack([rng.standard_normal(g.n_n) * 1e-3 for _ in range(nb)])
        for start in (None, x0):
            xs, reps, ms = g.pcg_batched(b, start, rel_tol=1e-10)
            assert ms > 0.0
            for m in range(nb):
                x1 = np.empty(g.n_n)
                r1 = _lib.SolveReportC()
                check(g.lib.mq_pcg_solve_host(g.ctx, dptr(b[m]), dptr(start[m]) if start is not None else None,
                                              dptr(x1), 1e-10, 0.0, 5000, 1, ctypes.byref(r1)))
                it, conv, rr, app = reps[m]
                assert conv and abs(it - r1.iterations) <= 1, (m, it, r1.iterations)
                assert rel(xs[m], x1) <= 1e-8
                assert rr <= 1e-10
        # budget exhaustion: every member reports its own non-convergence
        xs, reps, _ = g.pcg_batched(b, None, rel_tol=1e-14, max_iter=3)
        assert all(not c and it == 3 for it, c, _, _ in reps)
