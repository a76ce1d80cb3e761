"""Pin the CPU oracle against golden fixtures produced by the reference itself.

``tests/golden/make_golden.py`` ran the unmodified reference (mqsolve) on the
BASELINE configs' geometry; here the oracle repeats every step from the same
seeds.  Assembly, partition, SpMV and the conducting-block products must be
bit-identical; solver outputs must match to round-off (they are bit-identical
when numpy/OpenBLAS are the ones the fixtures were produced with).
"""

from __future__ import annotations

import hashlib
from pathlib import Path

import numpy as np
import pytest

from oracle import mq_oracle as O
from tests.conftest import oracle_model


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(np.asarray(a.shape, dtype=np.int64).tobytes())
        h.update(a.tobytes())
    return h.hexdigest()


def close(a, b, rtol=1e-12):
    a, b = np.asarray(a), np.asarray(b)
    return np.linalg.norm(a - b) <= rtol * max(np.linalg.norm(b), 1e-300)


def check_structure(golden, prefix, m):
    assert list(golden[f"{prefix}_n"]) == [m.n_c, m.n_n]
    assert sha(m.interior, m.cond, m.noncond) == str(golden[f"{prefix}_hash_partition"])
    assert sha(m.kn.indptr.astype(np.int64), m.kn.indices.astype(np.int64),
               m.kn.data) == str(golden[f"{prefix}_hash_kn"])
    assert sha(m.kcn.indptr.astype(np.int64), m.kcn.indices.astype(np.int64),
               m.kcn.data) == str(golden[f"{prefix}_hash_kcn"])
    assert sha(m.mc_diag) == str(golden[f"{prefix}_hash_mc"])
    assert sha(m.pattern) == str(golden[f"{prefix}_hash_pattern"])


def test_config0_structure_bit_exact(golden, oracle_c0):
    _, m = oracle_c0
    check_structure(golden, "c0", m)
    assert np.array_equal(m.noncond_global, golden["c0_noncond_global"])
    assert np.array_equal(m.cond_global, golden["c0_cond_global"])
    d, o = golden["c0_kn_diag_off"]
    assert np.all(m.kn.diagonal() == d)
    assert set(np.unique(np.abs(m.kn.data))) == {d, o}


def test_config1_structure_bit_exact(golden):
    _, m = oracle_model(1)
    check_structure(golden, "c1", m)
    assert list(golden["c1_n"]) == [45000, 717048]


def test_config0_pipeline(golden, oracle_c0):
    """Replay of make_golden.py's seeded sequence with the oracle."""
    spec, m = oracle_c0
    rng = np.random.default_rng(20250819)
    n_n, n_c = m.n_n, m.n_c
    x = rng.standard_normal(n_n)
    assert sha(x) == str(golden["c0_spmv_x__sha"])
    y = m.kn @ x
    assert np.array_equal(y, golden["c0_spmv_y"])
    _, mb = oracle_model(0, brauer=(3.8, 2.17, 396.2))
    st = rng.standard_normal(n_c) * 2e-4
    xc = rng.standard_normal(n_c)
    assert np.array_equal(st, golden["c0b_kc_state"])
    assert close(mb.kc_apply(st, xc), golden["c0b_kc_y"], 1e-14)
    assert np.array_equal(m.kc_apply(st, xc), golden["c0_kc_y"])
    assert np.array_equal(m.kcn.T @ xc, golden["c0_kcnt_y"])
    # PCG
    b = m.kn @ rng.standard_normal(n_n)
    x0 = rng.standard_normal(n_n) * 1e-3
    inv = O.jacobi_inverse(m.kn.diagonal())
    ra = O.pcg(m.kn_apply, b, rel_tol=1e-8, inv_diag=inv)
    rb = O.pcg(m.kn_apply, b, x0=x0, rel_tol=1e-8, inv_diag=inv)
    reps = golden["c0_pcg_reports"]
    assert ra.iterations == int(reps[0, 0]) and rb.iterations == int(reps[1, 0])
    assert close(ra.x, golden["c0_pcg_x_none"])
    assert abs(ra.rel - reps[0, 1]) <= 1e-6 * reps[0, 1]
    assert abs(np.linalg.norm(rb.x) - float(golden["c0_pcg_x_x0__norm"])) <= 1e-12 * np.linalg.norm(rb.x)
    rs = O.pcg(m.kn_apply, m.pattern, x0=np.zeros(n_n), rel_tol=1e-8, inv_diag=inv)
    assert rs.iterations == int(golden["c0_pcg_src_report"][0])
    # CSPE
    cache = O.SpeCache(n_n, m.kn_apply, max_cols=5, drop_tol=1e-8)
    seq = [O.pcg(m.kn_apply, m.kn @ rng.standard_normal(n_n), rel_tol=1e-8, inv_diag=inv).x
           for _ in range(6)]
    seq.append(seq[2] * 3.0)
    acc = [cache.insert(v) for v in seq]
    assert acc == list(golden["c0_cspe_accepted"])
    assert [cache.products, cache.accepted, cache.dropped, cache.evictions] == list(golden["c0_cspe_counts"])
    assert close(cache.G, golden["c0_cspe_galerkin"])
    rhs = m.kn @ rng.standard_normal(n_n)
    assert close(cache.project(rhs), golden["c0_cspe_x0"], 1e-10)
    # POD
    snap = O.Snapshots(n_n, n_pod=6, eps_pod=1e-4)
    for v in seq[:6] + [seq[0] + 1e-3 * seq[1], seq[3] * 0.5]:
        snap.push(v)
    x0p, kp, infop, appp = O.pod_start(snap, rhs, m.kn_apply)
    meta = golden["c0_pod_meta"]
    assert (kp, appp) == (int(meta[0]), int(meta[2]))
    assert abs(infop - meta[1]) <= 1e-12
    assert close(x0p, golden["c0_pod_x0"], 1e-8)


@pytest.mark.parametrize("strategy,nsteps", [("cspe", 100), ("pod", 30), ("previous", 30)])
def test_config0_transient(golden, oracle_c0, strategy, nsteps):
    spec, m = oracle_c0
    tr = O.run(m, O.sinusoid(50.0), spec.dt, nsteps, strategy=strategy, rel_tol=1e-8,
               max_cols=5, n_pod=20, eps_pod=1e-4)
    assert np.array_equal(np.array(tr.times), golden[f"c0_run_{strategy}_times"])
    norms = np.array([np.linalg.norm(a) for a in tr.a_c])
    ref = golden[f"c0_run_{strategy}_a_c_norms"]
    assert np.all(np.abs(norms - ref) <= 1e-10 * np.maximum(ref, 1e-300))
    assert close(tr.a_c[-1], golden[f"c0_run_{strategy}_a_c_final"], 1e-10)
    it = golden[f"c0_run_{strategy}_iters"]   # rows: [src mean, prev mean, cur]
    src = np.array(tr.iters[O.FAM_SOURCE])
    # row 0: initial recovery; row m: step m's source solve + recovery's
    assert it[0, 0] == src[0]
    assert np.array_equal(it[1:, 0], (src[1::2] + src[2::2]) / 2.0)
    assert np.array_equal(it[1:, 1], np.array(tr.iters[O.FAM_PREV]))
    assert np.array_equal(it[:, 2], np.array(tr.iters[O.FAM_CUR]))
    agg = golden[f"c0_run_{strategy}_agg"]
    assert int(agg[0]) == tr.steps
    assert int(agg[4]) == tr.pcg_applies
    assert int(agg[5]) == tr.maintenance


def test_config0_cfl(golden, oracle_c0):
    spec, m = oracle_c0
    op = O.SchurOracle(m, O.sinusoid(50.0), "cspe", 1e-8, 5000, 5)
    lam, dt, used = op.estimate_cfl()
    ref = golden["c0_cfl"]
    assert used == int(ref[2])
    assert abs(lam - ref[0]) <= 1e-10 * ref[0]
    assert abs(dt - spec.dt) <= 1e-6 * spec.dt   # SURVEY: 3.603515e-3


def test_config1_first_steps(golden):
    spec, m = oracle_model(1)
    tr = O.run(m, O.sinusoid(50.0), spec.dt, 2, strategy="cspe", rel_tol=1e-8, max_cols=5)
    it = golden["c1_run_cspe_iters"]
    assert np.array_equal(it[:, 2], np.array(tr.iters[O.FAM_CUR]))
    norms = np.array([np.linalg.norm(a) for a in tr.a_c])
    ref = golden["c1_run_cspe_a_c_norms"]
    assert np.all(np.abs(norms - ref) <= 1e-10 * np.maximum(ref, 1e-300))


@pytest.mark.parametrize("index", [0, 2])
def test_probe_b_matches_reference(golden, index):
    """model.py:415-425 probe_b and the default probe cells (model.py:562-566),
    against tests/golden/reference_probe.npz (tests/golden/make_golden_probe.py)."""
    from tests.golden.make_golden_probe import probe_states
    ref = np.load(Path(__file__).parent / "golden" / "reference_probe.npz")
    spec, m = oracle_model(index)
    cells = O.default_probe_cells(m, (spec.N,) * 3)
    assert np.array_equal(cells, ref[f"c{index}_probe_cells"])
    vals = [O.probe_b(m, O.full_interior(m, a_c, a_n), cells)
            for a_c, a_n in probe_states(index, m.n_c, m.n_n, golden)]
    assert np.array_equal(np.array(vals), ref[f"c{index}_probe_values"])
