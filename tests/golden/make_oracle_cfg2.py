"""Oracle reference data for configs[2] (128^3, two iron blocks, POD-30): the
first two explicit-Euler steps with recovery, run by the CPU oracle here
(minutes), stored compactly for the GPU parity test (norms, per-solve
iteration counts and 512 fixed sample entries of a_c and a_n per step).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_oracle_cfg2.py [--steps N]
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

OUT = Path(__file__).resolve().parent / "oracle_cfg2.npz"
STEPS = int(sys.argv[sys.argv.index("--steps") + 1]) if "--steps" in sys.argv else 2


def main():
    t0 = time.time()
    spec, m = oracle_model(2)
    print(f"assembled in {time.time() - t0:.0f} s (n_n {m.n_n}, n_c {m.n_c})", flush=True)
    tr = O.run(m, O.sinusoid(spec.freq), spec.dt, STEPS, strategy="pod", rel_tol=spec.rel_tol,
               n_pod=spec.n_pod, eps_pod=1e-4)
    rng = np.random.default_rng(7)
    ic = np.sort(rng.choice(m.n_c, 512, replace=False))
    inn = np.sort(rng.choice(m.n_n, 512, replace=False))
    out = {
        "idx_c": ic, "idx_n": inn,
        "a_c_norm": np.array([np.linalg.norm(a) for a in tr.a_c]),
        "a_n_norm": np.array([np.linalg.norm(a) for a in tr.a_n]),
        "a_c_sample": np.array([a[ic] for a in tr.a_c]),
        "a_n_sample": np.array([a[inn] for a in tr.a_n]),
        "iters_src": np.array(tr.iters[O.FAM_SOURCE]),
        "iters_prev": np.array(tr.iters[O.FAM_PREV]),
        "iters_cur": np.array(tr.iters[O.FAM_CUR]),
    }
    np.savez_compressed(OUT, **out)
    print(f"wrote {OUT} in {time.time() - t0:.0f} s", flush=True)


if __name__ == "__main__":
    main()
