"""Oracle reference data for configs[1] (64^3, Brauer iron): the first 20
explicit-Euler steps with recovery every step, with CSPE (k = 5) and with
POD-20, run by the CPU oracle here (minutes; the oracle is pinned to the
reference's own outputs by tests/test_oracle_golden.py), stored compactly for
the GPU parity test: per-step norms of a_c and a_n, per-solve iteration
counts, 512 fixed sample entries of a_c and a_n per step, the final a_c.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_oracle_cfg1.py
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_oracle_cfg1.py --long

--long: 100 CSPE steps into oracle_cfg1_long.npz (about 15 minutes here);
--long-pod: 60 POD-20 steps (every family's ring full and evicting) into
oracle_cfg1_pod_long.npz.
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import mq_oracle as O  # noqa: E402
from tests.conftest import oracle_model  # noqa: E402

LONG = "--long" in sys.argv
LONG_POD = "--long-pod" in sys.argv
OUT = Path(__file__).resolve().parent / ("oracle_cfg1_long.npz" if LONG else
                                         "oracle_cfg1_pod_long.npz" if LONG_POD else "oracle_cfg1.npz")
STEPS = 100 if LONG else (60 if LONG_POD else 20)
STRATEGIES = ("cspe",) if LONG else (("pod",) if LONG_POD else ("cspe", "pod"))


def main():
    t0 = time.time()
    spec, m = oracle_model(1)
    rng = np.random.default_rng(11)
    ic = np.sort(rng.choice(m.n_c, 512, replace=False))
    inn = np.sort(rng.choice(m.n_n, 512, replace=False))
    out = {"idx_c": ic, "idx_n": inn, "steps": np.array(STEPS), "dt": np.array(spec.dt)}
    for strat in STRATEGIES:
        tr = O.run(m, O.sinusoid(spec.freq), spec.dt, STEPS, strategy=strat, rel_tol=spec.rel_tol,
                   max_cols=5, n_pod=20, eps_pod=1e-4)
        out.update({
            f"{strat}_a_c_norm": np.array([np.linalg.norm(a) for a in tr.a_c]),
            f"{strat}_a_n_norm": np.array([np.linalg.norm(a) for a in tr.a_n]),
            f"{strat}_a_c_sample": np.array([a[ic] for a in tr.a_c]),
            f"{strat}_a_n_sample": np.array([a[inn] for a in tr.a_n]),
            f"{strat}_a_c_final": tr.a_c[-1],
            f"{strat}_iters_src": np.array(tr.iters[O.FAM_SOURCE]),
            f"{strat}_iters_prev": np.array(tr.iters[O.FAM_PREV]),
            f"{strat}_iters_cur": np.array(tr.iters[O.FAM_CUR]),
        })
        print(f"{strat}: {time.time() - t0:.0f} s", flush=True)
    np.savez_compressed(OUT, **out)
    print(f"wrote {OUT} in {time.time() - t0:.0f} s", flush=True)


if __name__ == "__main__":
    main()
