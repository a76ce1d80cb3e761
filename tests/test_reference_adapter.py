"""Problem.from_reference_model against the reference's own model objects
(CPU; needs the reference package, present in the build container only).

The device path consumes a Problem; a maintainer adapting an mqsolve Model
(INTEGRATION.md levels 1-2) goes through this adapter.  Checked here: the
adapted problem reproduces the reference model's partition, K_n
coefficients, source pattern and M_c through the oracle's assembly."""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

REF = Path("/root/reference/pkg/src")
pytestmark = pytest.mark.skipif(not REF.exists(), reason="reference package not available")


@pytest.fixture(scope="module")
def mq():
    sys.path.insert(0, str(REF))
    import mqsolve
    return mqsolve


@pytest.mark.parametrize("cells,linear", [(8, True), (10, False)])
def test_adapter_reproduces_reference_model(mq, cells, linear):
    from oracle import mq_oracle as O
    from paper_1611_06721_b200.device import Problem
    model = mq.builtin_model(cells=cells, linear=linear)
    prob = Problem.from_reference_model(model)
    assert prob.material.shape == (cells,) * 3
    assert prob.h == model.grid.h and prob.kappa == model.conductor.kappa
    kn = model.system.kn
    assert prob.kn_diag == kn.diagonal()[0]
    # the oracle assembled from the adapted problem has the reference's
    # partition, K_n and M_c
    om = O.assemble(prob.material, prob.h,
                    O.Conductor(prob.kappa, *prob.brauer), [])
    assert np.array_equal(om.interior[om.noncond], model.interior_edges[model.nonconducting])
    assert np.array_equal(om.interior[om.cond], model.interior_edges[model.conducting])
    dense_ref = np.zeros((kn.nrows, kn.nrows))
    rows = np.repeat(np.arange(kn.nrows), np.diff(kn.row_ptr))
    dense_ref[rows, kn.col_idx] = kn.values
    assert np.array_equal(om.kn.toarray(), dense_ref)
    assert np.array_equal(prob.pattern, np.asarray(model.system.source.pattern))
    mc = model.system.mc
    assert np.array_equal(om.mc_diag, mc.diagonal())
