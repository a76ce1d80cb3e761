"""Golden runs of the REFERENCE's SchurOperator options (schur.py:177-207,
244-250, 266-278): ``cache_source_solve=True``, ``projection_target=
"composed-coupling"`` and ``strategy=<StartVectorStrategy instance>``.

Run in the build container, where /root/reference exists:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_options.py

Config 0 (same shim as make_golden.py), CSPE k = 5, 20 steps with an output
row after every step and the reference's own B probe.  Stored per run: the
TransientResult columns and the trace CSV bytes (bench.py:341-357).
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

OUT = Path(__file__).resolve().parent
NSTEPS = 20


def main():
    sys.path.insert(0, str(OUT))
    from make_golden import reference_model
    from mqsolve import PcgConfig, Preconditioner, run_explicit
    from mqsolve.bench import trace_bytes
    from mqsolve.startvec import make_strategy

    spec, m, _ = reference_model(0)
    dt = spec.dt
    out = {"dt": np.array(dt), "nsteps": np.array(NSTEPS)}
    runs = {
        "cache_src": dict(strategy="cspe", cache_source_solve=True),
        "composed": dict(strategy="cspe", projection_target="composed-coupling"),
        # a strategy instance (isinstance StartVectorStrategy, schur.py:198-199);
        # the operator it is handed is the model's K_n product
        "instance": dict(strategy=make_strategy("cspe", m.n_n, lambda x: m.system.kn.to_scipy() @ x,
                                                max_cols=5, drop_tol=1e-8)),
    }
    for key, kw in runs.items():
        t0 = time.time()
        res = run_explicit(m.system, t_end=NSTEPS * dt, dt=dt, pcg=PcgConfig(rel_tol=1e-8, max_iter=5000),
                           preconditioner=Preconditioner.JACOBI, output_period=dt * (1 - 1e-3),
                           probe=m.probe_callable(), max_cols=5, **kw)
        for col in ("times", "probe_b", "iters_src", "iters_cpl_prev", "iters_cpl_cur",
                    "basis_cols", "pod_k", "pod_info", "final_a_c", "final_a_n"):
            out[f"{key}_{col}"] = np.asarray(getattr(res, col))
        out[f"{key}_trace"] = np.frombuffer(trace_bytes(res), dtype=np.uint8)
        out[f"{key}_solves"] = np.array([res.aggregates["solves"][f] for f in
                                         ("source", "coupling_current", "coupling_previous")])
        print(f"{key}: {res.n_rows} rows in {time.time() - t0:.1f} s; src iters {res.iters_src[:6]}", flush=True)
    np.savez_compressed(OUT / "reference_options.npz", **out)
    print("wrote", OUT / "reference_options.npz")


if __name__ == "__main__":
    main()
