"""Per-step A-field fixtures for the config-scale parity tests.

Runs the CPU oracle (pinned to the reference by tests/test_oracle_golden.py)
over the first steps of a BASELINE config, recovery every step (4 solves per
step), and stores for every output row t = 0..steps:
the exact norm of the A-field (a_c, a_n) and its CountSketch
(tests/fieldcheck.py), per-solve iteration counts, the oracle's own wall time
per step, and the full field at the last step (a_c only for 128^3).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_oracle_fields.py CASE

CASE: cfg1_cspe (100 steps), cfg1_pod (60 steps, POD-20), cfg2 (25 steps,
128^3 POD-30), cfg3_m255 (ensemble member 255, 20 steps).
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import mq_oracle as O  # noqa: E402
from paper_1611_06721_b200 import configs as C  # noqa: E402
from tests import fieldcheck as F  # noqa: E402
from tests.conftest import oracle_model  # noqa: E402

CASES = {
    "cfg1_cspe": dict(index=1, steps=100, strategy="cspe"),
    "cfg1_pod": dict(index=1, steps=60, strategy="pod", n_pod=20),
    "cfg2": dict(index=2, steps=25, strategy="pod", n_pod=30),
    "cfg3_m255": dict(index=3, steps=20, strategy="cspe", member=255),
}


class TimedOp(O.SchurOracle):
    """SchurOracle that stamps the wall time at the end of every recovery."""
    stamps: list

    def recover(self, a_c, t):
        out = super().recover(a_c, t)
        self.stamps.append(time.perf_counter())
        return out


def main(case: str):
    c = CASES[case]
    t0 = time.time()
    kw = {}
    dt = None
    if "member" in c:
        j, k = C.ensemble_factors(256, 0)
        kw = dict(j_scale=float(j[c["member"]]), kappa_scale=float(k[c["member"]]))
        dt = C.config_spec(3).dt * kw["kappa_scale"]
    spec, m = oracle_model(c["index"], **kw)
    dt = spec.dt if dt is None else dt
    print(f"{case}: assembled in {time.time() - t0:.0f} s (n_n {m.n_n}, n_c {m.n_c}), dt {dt!r}",
          flush=True)
    stamps: list = []
    orig = O.SchurOracle
    TimedOp.stamps = stamps
    O.SchurOracle = TimedOp
    try:
        tr = O.run(m, O.sinusoid(spec.freq), dt, c["steps"], strategy=c["strategy"],
                   rel_tol=spec.rel_tol, max_cols=5, n_pod=c.get("n_pod", 10), eps_pod=1e-4)
    finally:
        O.SchurOracle = orig
    plan = F.sketch_plan(m.n_c + m.n_n)
    fields = [F.field_of(a, b) for a, b in zip(tr.a_c, tr.a_n)]
    out = {
        "case": np.array(case), "steps": np.array(c["steps"]), "dt": np.array(dt),
        "n_c": np.array(m.n_c), "n_n": np.array(m.n_n),
        "norm": np.array([np.linalg.norm(f) for f in fields]),
        "sketch": np.array([F.sketch(f, plan) for f in fields]),
        "iters_src": np.array(tr.iters[O.FAM_SOURCE]),
        "iters_prev": np.array(tr.iters[O.FAM_PREV]),
        "iters_cur": np.array(tr.iters[O.FAM_CUR]),
        "step_seconds": np.diff(np.array(stamps)),
        "a_c_final": tr.a_c[-1],
    }
    if c["index"] != 2:
        out["a_n_final"] = tr.a_n[-1]
    dst = Path(__file__).resolve().parent / f"fields_{case}.npz"
    np.savez_compressed(dst, **out)
    print(f"wrote {dst} in {time.time() - t0:.0f} s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1])
