"""Golden trace rows from the REFERENCE's run_explicit (schur.py:474-607).

Run in the build container, where /root/reference exists:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_trace.py

Config 0 (same shim as make_golden.py) with the reference's own B probe
(model.probe_callable), strategies cspe (100 steps), pod (30 steps, n_pod 20)
and previous (30 steps) with an output row after every step, plus cspe and
pod with an output row every third step (windows of three Euler steps).
Stored per run: every TransientResult column, the aggregates the device twin
reports, and the trace CSV bytes of the reference's bench.trace_bytes
(bench.py:341-357).
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

OUT = Path(__file__).resolve().parent
RUNS = (("cspe", 100, 1), ("pod", 30, 1), ("previous", 30, 1), ("cspe", 30, 3), ("pod", 30, 3))


def main():
    sys.path.insert(0, str(OUT))
    from make_golden import reference_model
    from mqsolve import PcgConfig, Preconditioner, run_explicit
    from mqsolve.bench import trace_bytes

    spec, m, _ = reference_model(0)
    dt = spec.dt
    out = {"dt": np.array(dt)}
    for strat, nsteps, every in RUNS:
        t0 = time.time()
        res = run_explicit(m.system, t_end=nsteps * dt, dt=dt, strategy=strat,
                           pcg=PcgConfig(rel_tol=1e-8, max_iter=5000),
                           preconditioner=Preconditioner.JACOBI,
                           output_period=every * dt * (1 - 1e-3), probe=m.probe_callable(),
                           max_cols=5, n_pod=20, eps_pod=1e-4)
        key = f"{strat}_{nsteps}_{every}"
        for col in ("times", "probe_b", "iters_src", "iters_cpl_prev", "iters_cpl_cur",
                    "basis_cols", "pod_k", "pod_info", "final_a_c", "final_a_n"):
            out[f"{key}_{col}"] = np.asarray(getattr(res, col))
        agg = res.aggregates
        out[f"{key}_agg"] = np.array([agg["steps"], agg["pcg_applies"], agg["maintenance_applies"],
                                      agg["min_pod_info"], agg["max_basis_cols"]])
        out[f"{key}_trace"] = np.frombuffer(trace_bytes(res), dtype=np.uint8)
        print(f"{key}: {res.n_rows} rows in {time.time() - t0:.1f} s; basis {res.basis_cols[:8]}, "
              f"pod_k {res.pod_k[:8]}", flush=True)
    np.savez_compressed(OUT / "reference_trace.npz", **out)
    print("wrote", OUT / "reference_trace.npz")


if __name__ == "__main__":
    main()
