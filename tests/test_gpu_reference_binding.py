"""The reference's OWN time stepper driving the device path.

``mqsolve.run_explicit`` (mq/schur.py:474-607), unmodified, on config 0 with
the reference's B probe, through the bindings of
:mod:`paper_1611_06721_b200.refbind`:

* section 2: ``mqsolve.schur.pcg_solve`` rebound, so every K_n solve of the
  reference's ``SchurOperator`` is a device PCG;
* section 1: a :class:`DeviceStrategy` instance injected as ``strategy=``
  (the reference runs its own PCG, the start vectors come from the GPU);
* both at once.

Each run is compared with the reference's own run without any binding
(tests/golden/reference_trace.npz): the trace rows (times, basis_cols, pod_k
exact; iteration means +-1; B_probe within the field bar) and the final
A-field within 1e-8 relative L2.

The reference is imported from ``baseline/_ref`` (``pip install --target``
of /root/reference, made in the build container; git-ignored, shipped to the
GPU box with the snapshot) or from /root/reference itself; without either
the module is skipped.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
CANDIDATES = [ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")]
REF = next((p for p in CANDIDATES if (p / "mqsolve").exists()), None)

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(REF is None, reason="reference package not installed (baseline/_ref)")]

REL_FIELD = 1e-8
RUNS = [("cspe", 100), ("pod", 30), ("previous", 30)]


@pytest.fixture(scope="module")
def ref(gpu_ok):
    sys.path.insert(0, str(REF))
    import mqsolve
    import mqsolve.schur as S
    import mqsolve.startvec  # noqa: F401
    from tests.refmodel import reference_model
    spec, model, _ = reference_model(0)
    gold = np.load(ROOT / "tests" / "golden" / "reference_trace.npz")
    return mqsolve, S, spec, model, gold


def _run(mqsolve, model, dt, strategy, nsteps):
    return mqsolve.run_explicit(model.system, t_end=nsteps * dt, dt=dt, strategy=strategy,
                                pcg=mqsolve.PcgConfig(rel_tol=1e-8, max_iter=5000),
                                preconditioner=mqsolve.Preconditioner.JACOBI,
                                output_period=dt * (1 - 1e-3), probe=model.probe_callable(),
                                max_cols=5, n_pod=20, eps_pod=1e-4)


def _check(res, gold, key):
    assert np.array_equal(res.times, gold[f"{key}_times"])
    assert np.array_equal(res.basis_cols, gold[f"{key}_basis_cols"])
    assert np.array_equal(res.pod_k, gold[f"{key}_pod_k"])
    assert np.max(np.abs(res.pod_info - gold[f"{key}_pod_info"])) <= 20 * REL_FIELD
    for col in ("iters_src", "iters_cpl_prev", "iters_cpl_cur"):
        assert np.max(np.abs(getattr(res, col) - gold[f"{key}_{col}"])) <= 1.0, col
    b = gold[f"{key}_probe_b"]
    assert np.max(np.abs(res.probe_b - b)) <= REL_FIELD * np.abs(b).max()
    a = np.concatenate([res.final_a_c, res.final_a_n])
    a_ref = np.concatenate([gold[f"{key}_final_a_c"], gold[f"{key}_final_a_n"]])
    assert np.linalg.norm(a - a_ref) <= REL_FIELD * np.linalg.norm(a_ref)


@pytest.mark.parametrize("strategy,nsteps", RUNS)
def test_reference_loop_with_device_pcg(ref, strategy, nsteps):
    """the reference's loop, every K_n solve on the GPU."""
    from paper_1611_06721_b200.refbind import bind_pcg, grid_for_model
    mqsolve, S, spec, model, gold = ref
    dt = float(gold["dt"])
    grid = grid_for_model(model)
    try:
        with bind_pcg(S, grid) as binding:
            res = _run(mqsolve, model, dt, strategy, nsteps)
        assert S.pcg_solve is binding.reference_pcg          # restored
        # every inner solve of the run went to the device: 2 per step + 2 per row
        assert binding.device_solves == 2 * nsteps + 2 * res.n_rows
        assert res.aggregates["pcg_applies"] == binding.kn.count
        _check(res, gold, f"{strategy}_{nsteps}_1")
    finally:
        grid.close()


@pytest.mark.parametrize("strategy,nsteps", [("cspe", 100), ("pod", 30)])
def test_reference_loop_with_device_strategy(ref, strategy, nsteps):
    """a DeviceStrategy injected into the reference's loop."""
    from paper_1611_06721_b200.refbind import device_strategy, grid_for_model
    mqsolve, S, spec, model, gold = ref
    dt = float(gold["dt"])
    grid = grid_for_model(model)
    try:
        strat = device_strategy(grid, strategy, base=mqsolve.startvec.StartVectorStrategy, max_cols=5,
                                n_pod=20, eps_pod=1e-4, drop_tol=1e-8)
        assert isinstance(strat, mqsolve.startvec.StartVectorStrategy)
        res = _run(mqsolve, model, dt, strat, nsteps)
        assert res.aggregates["strategy"] == strategy
        _check(res, gold, f"{strategy}_{nsteps}_1")
    finally:
        grid.close()


def test_reference_loop_with_both_bindings(ref):
    """Sections 1 and 2 together: start vectors and solves on the GPU, the
    loop, the Euler update and the recovery in the reference."""
    from paper_1611_06721_b200.refbind import bind_pcg, device_strategy, grid_for_model
    mqsolve, S, spec, model, gold = ref
    dt = float(gold["dt"])
    grid = grid_for_model(model)
    try:
        strat = device_strategy(grid, "cspe", base=mqsolve.startvec.StartVectorStrategy, max_cols=5,
                                drop_tol=1e-8)
        with bind_pcg(S, grid):
            res = _run(mqsolve, model, dt, strat, 100)
        _check(res, gold, "cspe_100_1")
        assert res.aggregates["max_basis_cols"] == 5
    finally:
        grid.close()
