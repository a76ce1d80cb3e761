"""Manifest loader of the CSR-system path on the CPU:
the blocks, pattern and waveform of a model exported by the reference's
export_model (model.py:640-689) equal what the reference's load_model
(bench.py:228-313) returns (tests/golden/make_manifest_fixture.py), and the
loader rejects what the reference rejects.  No GPU needed."""
import json
import math
import shutil
from pathlib import Path

import numpy as np
import pytest

GOLD = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def ref():
    return np.load(GOLD / "manifest_c6_ref.npz")


def test_load_manifest_matches_reference(ref):
    from paper_1611_06721_b200.csrsys import load_manifest
    s = load_manifest(GOLD / "manifest_c6")
    for name, blk in (("m_c", s.mc), ("k_c", s.kc), ("k_cn", s.kcn), ("k_n", s.kn)):
        assert np.array_equal(blk.indptr, ref[f"{name}_rp"]), name
        assert np.array_equal(blk.indices, ref[f"{name}_ci"]), name
        assert np.array_equal(blk.data, ref[f"{name}_va"]), name
    assert np.array_equal(s.pattern, ref["pattern"])
    assert (s.n_c, s.n_n) == (96, 354)
    for t, w in zip(ref["ramp_t"], ref["ramp_w"]):
        assert s.waveform(float(t)) == w


def _copy(tmp_path):
    d = tmp_path / "m"
    shutil.copytree(GOLD / "manifest_c6", d)
    return d, json.loads((d / "manifest.json").read_text())


def _write(d, mf):
    (d / "manifest.json").write_text(json.dumps(mf))


def test_load_manifest_sinusoid_kind(tmp_path):
    from paper_1611_06721_b200.csrsys import load_manifest
    d, mf = _copy(tmp_path)
    mf["waveform"] = {"kind": "sinusoid", "frequency": 50.0}
    _write(d, mf)
    s = load_manifest(d)
    for t in (0.0, 1e-3, 7.3e-3):
        assert s.waveform(t) == math.sin(2.0 * math.pi * 50.0 * t)


@pytest.mark.parametrize("case", ["missing", "format", "kind", "block_file", "pattern_len", "asym"])
def test_load_manifest_rejects(tmp_path, case):
    from paper_1611_06721_b200.csrsys import ConfigError, load_manifest
    d, mf = _copy(tmp_path)
    if case == "missing":
        (d / "manifest.json").unlink()
    elif case == "format":
        mf["format"] = "other"
        _write(d, mf)
    elif case == "kind":
        mf["waveform"] = {"kind": "square"}
        _write(d, mf)
    elif case == "block_file":
        (d / mf["blocks"]["k_n"]["file"]).unlink()
    elif case == "pattern_len":
        import scipy.io
        scipy.io.mmwrite(str(d / mf["blocks"]["source_pattern"]["file"]), np.ones((5, 1)), field="real")
    elif case == "asym":
        import scipy.io
        import scipy.sparse as sp
        f = d / mf["blocks"]["k_n"]["file"]
        k = sp.csr_matrix(scipy.io.mmread(str(f)))
        k[0, 1] = k[0, 1] + 1.0
        scipy.io.mmwrite(str(f), k, symmetry="general")
    with pytest.raises(ConfigError):
        load_manifest(d)


def test_builtin_section_rebuilds_and_checks_pattern(tmp_path):
    """bench.py:283-306 on the host side: the builtin section rebuilds the
    model (configs.builtin_problem, model.py:582-622) and a stored pattern
    that disagrees with it is refused."""
    from paper_1611_06721_b200.csrsys import ConfigError, is_diagonal, load_manifest
    d, mf = _copy(tmp_path / "a")
    mf["builtin"] = {"cells": 6, "h": 5e-3, "kappa": 5e6, "brauer": [49.4, 1.46, 520.6], "amps": 50000.0,
                     "tau": 0.5, "linear": False}
    (d / "manifest.json").write_text(json.dumps(mf))
    s = load_manifest(d)
    assert s.builtin is not None and s.builtin.material.shape == (6, 6, 6)
    assert np.array_equal(s.builtin.pattern, s.pattern)
    assert is_diagonal(s.mc)
    mf["builtin"]["amps"] = 40000.0
    (d / "manifest.json").write_text(json.dumps(mf))
    with pytest.raises(ConfigError, match="pattern"):
        load_manifest(d)
