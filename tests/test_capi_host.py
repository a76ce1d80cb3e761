"""CPU tests: the C-ABI library loads and exports every declared symbol, and
the host-side logic (config geometry, source pattern, step schedule) agrees
with the oracle.  No device compute here."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import mq_oracle as O
from paper_1611_06721_b200 import _lib
from paper_1611_06721_b200 import configs as C
from paper_1611_06721_b200.schur import step_times


@pytest.fixture(scope="module")
def lib():
    from paper_1611_06721_b200 import build
    build.build()
    return _lib.load()


def test_library_exports_every_header_symbol(lib):
    declared = _lib.header_symbols()
    assert len(declared) >= 40
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    # and the ctypes table binds exactly the header's entry points
    assert sorted(_lib.SIGNATURES) == declared


def test_no_gpu_calls_fail_loudly_without_device(lib):
    if _lib.device_count() > 0:
        pytest.skip("a GPU is visible")
    from paper_1611_06721_b200.device import DeviceGrid
    with pytest.raises(Exception):
        DeviceGrid(C.make_problem(0))


def test_missing_library_raises(tmp_path):
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _lib.load(tmp_path / "absent.so")


@pytest.mark.parametrize("index", [0, 1])
def test_config_geometry_matches_oracle(index):
    spec = C.config_spec(index)
    mat = C.material_map(spec)
    loops = C.coil_loops(spec.N, spec.J)
    m = O.assemble(mat, spec.h, O.Conductor(spec.kappa, *spec.brauer),
                   [O.Loop(lp.i0, lp.i1, lp.j0, lp.j1, lp.k0, lp.amps) for lp in loops])
    flag, _ = C.noncond_positions(mat)
    assert np.array_equal(np.flatnonzero(flag), m.noncond_global)
    assert np.array_equal(C.source_pattern(mat, loops), m.pattern)
    expect = {0: (882, 9918), 1: (45000, 717048)}[index]
    assert (m.n_c, m.n_n) == expect


def test_config_sizes_large():
    """Configs 2 and 4 partition sizes without assembling."""
    for index, (nc, nn) in ((2, (90000, 6103536)),):
        spec = C.config_spec(index)
        flag, _ = C.noncond_positions(C.material_map(spec))
        assert int(flag.sum()) == nn
        N = spec.N
        interior = 3 * N * (N - 1) ** 2
        assert interior - nn == nc


def test_coil_loops_are_closed_and_clear():
    for index in (0, 1, 2):
        spec = C.config_spec(index)
        mat = C.material_map(spec)
        loops = C.coil_loops(spec.N, spec.J)
        s = spec.N // 16
        assert len(loops) == (4 * s + 1) * (2 * s + 1)
        pat = C.source_pattern(mat, loops)
        assert np.count_nonzero(pat) > 0


def test_step_schedule_matches_reference_loop():
    """schur.py:546-572 step count and output trigger."""
    dt = 3.603515e-3
    dts, outs = step_times(100 * dt, dt, dt * (1 - 1e-3))
    assert len(dts) == 100 and all(outs)
    dts, outs = step_times(1e-2, 1e-3, 2e-3)
    assert len(dts) == 10 and sum(outs) == 5
    dts, outs = step_times(1.05e-2, 1e-3, 1e-3)
    assert len(dts) == 11 and abs(dts[-1] - 5e-4) < 1e-15


def test_ensemble_factors_deterministic():
    j1, k1 = C.ensemble_factors(256, 7)
    j2, k2 = C.ensemble_factors(256, 7)
    assert np.array_equal(j1, j2) and np.array_equal(k1, k2)
    assert j1.min() >= 0.8 and j1.max() <= 1.2
