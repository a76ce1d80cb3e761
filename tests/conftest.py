"""Shared fixtures for the mq-b200 tests.

``-m "not gpu"`` tests run on CPU (oracle vs golden fixtures, host logic, the
C-ABI library's exported symbols).  ``-m gpu`` tests are the parity tests
proper: they call the CUDA path through the C ABI and compare it with the
oracle (``oracle/mq_oracle.py``) on the same seeded inputs.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden" / "reference_golden.npz"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libmq_b200.so")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def golden():
    return dict(np.load(GOLDEN, allow_pickle=False))


@pytest.fixture
def rng():
    return np.random.default_rng(20250819)


def oracle_model(index: int, brauer=None, j_scale=1.0, kappa_scale=1.0):
    """Oracle assembly of a BASELINE config (same recipe as the product)."""
    from oracle import mq_oracle as O
    from paper_1611_06721_b200 import configs as C
    spec = C.config_spec(index)
    mat = C.material_map(spec)
    loops = C.coil_loops(spec.N, spec.J * j_scale)
    k1, k2, k3 = brauer or spec.brauer
    m = O.assemble(mat, spec.h, O.Conductor(spec.kappa * kappa_scale, k1, k2, k3),
                   [O.Loop(lp.i0, lp.i1, lp.j0, lp.j1, lp.k0, lp.amps) for lp in loops])
    return spec, m


@pytest.fixture(scope="session")
def oracle_c0():
    return oracle_model(0)


@pytest.fixture(scope="session")
def gpu_ok():
    """Skip-free guard: GPU tests must fail loudly when the library is missing."""
    from paper_1611_06721_b200 import _lib
    _lib.load()
    assert _lib.device_count() >= 1, "no CUDA device visible"
    return True
