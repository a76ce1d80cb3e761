"""Generate golden fixtures by running the REFERENCE (mqsolve) itself.

Run in the build container, where /root/reference exists:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports the unmodified reference from /root/reference/pkg/src and records
its outputs on the BASELINE configs' geometry (SURVEY 8(d) recipe: the
annular coil as a sum of closed loops, sinusoidal waveform), so that the
oracle (``oracle/mq_oracle.py``) can be pinned against the reference on the
GPU box, where /root/reference does not exist.  Only small arrays are kept.
"""

from __future__ import annotations

import hashlib
import math
import sys
import time
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(REF))
sys.path.insert(0, str(ROOT))

import mqsolve  # noqa: E402
import mqsolve.model as M  # noqa: E402
from mqsolve import (CsrMatrix, Excitation, GridSpec, Material, PcgConfig,  # noqa: E402
                     Preconditioner, ScaledPatternSource, SnapshotBuffer, SubspaceCache,
                     pcg_solve, pod_start_vector, run_explicit)

from paper_1611_06721_b200 import configs as C  # noqa: E402  (geometry recipe only)

OUT = Path(__file__).resolve().parent
SEED = 20250819


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(np.asarray(a.shape, dtype=np.int64).tobytes())
        h.update(a.tobytes())
    return h.hexdigest()


from tests.refmodel import reference_model  # noqa: E402,F401  (shared with the binding tests)


def put(out, name, arr, full=True):
    """Store sha256 + 2-norm always, the values only when ``full``."""
    arr = np.asarray(arr)
    out[f"{name}__sha"] = np.array(sha(arr))
    if arr.dtype.kind == "f":
        out[f"{name}__norm"] = np.array(float(np.linalg.norm(arr)))
    if full:
        out[name] = arr


def structure(prefix, model, pattern, out, full=True):
    sysm = model.system
    kn, kcn = sysm.kn, sysm.kcn
    out[f"{prefix}_n"] = np.array([model.n_c, model.n_n])
    out[f"{prefix}_hash_partition"] = sha(model.interior_edges, model.conducting, model.nonconducting)
    out[f"{prefix}_hash_kn"] = sha(kn.row_ptr, kn.col_idx, kn.values)
    out[f"{prefix}_hash_kcn"] = sha(kcn.row_ptr, kcn.col_idx, kcn.values)
    out[f"{prefix}_hash_mc"] = sha(sysm.mc.diagonal())
    out[f"{prefix}_hash_pattern"] = sha(pattern)
    out[f"{prefix}_kn_diag_off"] = np.array([np.unique(kn.diagonal())[0],
                                             np.unique(np.abs(kn.values))[0]])
    if full:
        out[f"{prefix}_noncond_global"] = model.interior_edges[model.nonconducting]
        out[f"{prefix}_cond_global"] = model.interior_edges[model.conducting]
        out[f"{prefix}_mc_diag"] = sysm.mc.diagonal()
        out[f"{prefix}_pattern"] = pattern


def main():
    t0 = time.time()
    out = {}
    rng = np.random.default_rng(SEED)

    # ---- config 0 (16^3, linear iron): structure, kernels, solver pieces ----
    spec0, m0, pat0 = reference_model(0)
    structure("c0", m0, pat0, out)
    kn0 = m0.system.kn
    n_n, n_c = m0.n_n, m0.n_c
    x = rng.standard_normal(n_n)
    put(out, "c0_spmv_x", x, False)
    put(out, "c0_spmv_y", kn0.to_scipy() @ x)
    # Brauer K_c on the config-0 geometry with the config-1 material
    _, m0b, _ = reference_model(0, brauer=C.BRAUER_IRON)
    st = rng.standard_normal(n_c) * 2e-4
    xc = rng.standard_normal(n_c)
    out["c0b_kc_state"] = st
    out["c0b_kc_x"] = xc
    out["c0b_kc_y"] = m0b.system.kc_apply(st, xc)
    out["c0_kc_y"] = m0.system.kc_apply(st, xc)
    out["c0_kcnt_y"] = m0.system.kcn.to_scipy().T @ xc
    # PCG: consistent rhs, Jacobi, x0 None and x0 given
    b = kn0.to_scipy() @ rng.standard_normal(n_n)
    x0 = rng.standard_normal(n_n) * 1e-3
    cfg = PcgConfig(rel_tol=1e-8, max_iter=5000, preconditioner=Preconditioner.JACOBI)
    xa, ra = pcg_solve(kn0, b, config=cfg)
    xb, rb = pcg_solve(kn0, b, x0=x0, config=cfg)
    put(out, "c0_pcg_b", b, False)
    put(out, "c0_pcg_x0", x0, False)
    put(out, "c0_pcg_x_none", xa)
    put(out, "c0_pcg_x_x0", xb, False)
    out["c0_pcg_reports"] = np.array([[ra.iterations, ra.final_rel_residual, ra.converged],
                                      [rb.iterations, rb.final_rel_residual, rb.converged]])
    # source solve with the pattern (a realistic inner solve)
    xs, rs = pcg_solve(kn0, pat0, x0=np.zeros(n_n), config=cfg)
    put(out, "c0_pcg_src_x", xs, False)
    out["c0_pcg_src_report"] = np.array([rs.iterations, rs.final_rel_residual])
    # CSPE cache: 7 inserts into max_cols=5, then a projection
    op = lambda v: kn0.to_scipy() @ v  # noqa: E731
    cache = SubspaceCache(n_n, op, max_cols=5, drop_tol=1e-8)
    seq = [pcg_solve(kn0, kn0.to_scipy() @ rng.standard_normal(n_n), config=cfg)[0]
           for _ in range(6)]
    seq.append(seq[2] * 3.0)  # dependent: dropped
    acc = [cache.insert(v) for v in seq]
    rhs = kn0.to_scipy() @ rng.standard_normal(n_n)
    put(out, "c0_cspe_seq", np.column_stack(seq), False)
    out["c0_cspe_accepted"] = np.array(acc)
    put(out, "c0_cspe_basis", cache.basis, False)
    put(out, "c0_cspe_products", cache.cached_products, False)
    out["c0_cspe_galerkin"] = cache.galerkin
    out["c0_cspe_counts"] = np.array([cache.products_computed, cache.columns_accepted,
                                      cache.columns_dropped, cache.evictions])
    put(out, "c0_cspe_rhs", rhs, False)
    put(out, "c0_cspe_x0", cache.project(rhs))
    # POD: ring of 6, 8 pushes, projection
    buf = SnapshotBuffer(n_n, n_pod=6, eps_pod=1e-4)
    for v in seq[:6] + [seq[0] + 1e-3 * seq[1], seq[3] * 0.5]:
        buf.push(v)
    x0p, kp, infop, appp = pod_start_vector(buf, rhs, op)
    put(out, "c0_pod_snapshots", buf.matrix(), False)
    put(out, "c0_pod_x0", x0p)
    out["c0_pod_meta"] = np.array([kp, infop, appp])

    # ---- config-0 transients, output every step ------------------------------
    dt0 = spec0.dt
    for strat, nsteps in (("cspe", 100), ("pod", 30), ("previous", 30)):
        states = []

        def probe(a_c, a_n, t):
            states.append((t, a_c.copy(), a_n.copy()))
            return 0.0

        tr = time.time()
        res = run_explicit(m0.system, t_end=nsteps * dt0, dt=dt0, strategy=strat,
                           pcg=PcgConfig(rel_tol=1e-8, max_iter=5000),
                           preconditioner=Preconditioner.JACOBI,
                           output_period=dt0 * (1 - 1e-3), probe=probe, max_cols=5,
                           n_pod=20, eps_pod=1e-4)
        agg = res.aggregates
        out[f"c0_run_{strat}_times"] = np.array([s[0] for s in states])
        put(out, f"c0_run_{strat}_a_c", np.array([s[1] for s in states]), False)
        out[f"c0_run_{strat}_a_c_norms"] = np.array([np.linalg.norm(s[1]) for s in states])
        out[f"c0_run_{strat}_a_c_final"] = states[-1][1]
        put(out, f"c0_run_{strat}_a_n_final", states[-1][2], False)
        out[f"c0_run_{strat}_a_n_norms"] = np.array([np.linalg.norm(s[2]) for s in states])
        out[f"c0_run_{strat}_iters"] = np.stack([res.iters_src, res.iters_cpl_prev,
                                                 res.iters_cpl_cur], axis=1)
        out[f"c0_run_{strat}_agg"] = np.array([
            agg["steps"], agg["iterations"]["source"], agg["iterations"]["coupling_previous"],
            agg["iterations"]["coupling_current"], agg["pcg_applies"],
            agg["maintenance_applies"], agg["min_pod_info"], agg["max_basis_cols"]])
        print(f"config 0 {strat}: {nsteps} steps in {time.time() - tr:.1f}s, "
              f"iters {agg['iterations']}", flush=True)

    # ---- config 0 CFL estimate (schur.py:327-376) ----------------------------
    from mqsolve import SchurOperator, estimate_cfl
    opx = SchurOperator(m0.system, pcg=PcgConfig(rel_tol=1e-8, max_iter=5000),
                        strategy="cspe", preconditioner=Preconditioner.JACOBI, max_cols=5)
    est = estimate_cfl(opx, safety=0.9, seed=42)
    out["c0_cfl"] = np.array([est.lambda_max, est.dt_max, est.power_iters])
    print("config 0 CFL", est, flush=True)

    # ---- config 1 (64^3, Brauer): structure + first 2 steps -----------------
    spec1, m1, pat1 = reference_model(1)
    structure("c1", m1, pat1, out, full=False)
    states = []

    def probe1(a_c, a_n, t):
        states.append((t, a_c.copy(), np.linalg.norm(a_n)))
        return 0.0

    tr = time.time()
    res = run_explicit(m1.system, t_end=2 * spec1.dt, dt=spec1.dt, strategy="cspe",
                       pcg=PcgConfig(rel_tol=1e-8, max_iter=5000),
                       preconditioner=Preconditioner.JACOBI,
                       output_period=spec1.dt * (1 - 1e-3), probe=probe1, max_cols=5)
    put(out, "c1_run_cspe_a_c", np.array([s[1] for s in states]), False)
    out["c1_run_cspe_a_c_norms"] = np.array([np.linalg.norm(s[1]) for s in states])
    out["c1_run_cspe_a_n_norms"] = np.array([s[2] for s in states])
    out["c1_run_cspe_iters"] = np.stack([res.iters_src, res.iters_cpl_prev,
                                         res.iters_cpl_cur], axis=1)
    print(f"config 1 cspe 2 steps in {time.time() - tr:.1f}s", flush=True)

    out["meta"] = np.array([f"reference mqsolve {mqsolve.__version__}",
                            f"numpy {np.__version__}",
                            f"scipy {__import__('scipy').__version__}"])
    np.savez_compressed(OUT / "reference_golden.npz", **out)
    print(f"wrote {OUT / 'reference_golden.npz'} in {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
