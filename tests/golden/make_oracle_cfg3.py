"""Oracle reference data for a configs[3] ensemble member (64^3, J and kappa
factors from the ensemble seed, dt scaled with kappa): member 255, the first
20 steps with CSPE k = 5, stored compactly like make_oracle_cfg1.py.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_oracle_cfg3.py
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
from tests.conftest import oracle_model  # noqa: E402

OUT = Path(__file__).resolve().parent / "oracle_cfg3_member255.npz"
MEMBER, STEPS = 255, 20


def main():
    t0 = time.time()
    j, k = C.ensemble_factors(256, 0)
    jf, kf = float(j[MEMBER]), float(k[MEMBER])
    dt = C.config_spec(3).dt * kf
    spec, m = oracle_model(3, j_scale=jf, kappa_scale=kf)
    tr = O.run(m, O.sinusoid(spec.freq), dt, STEPS, strategy="cspe", rel_tol=1e-8, max_cols=5)
    rng = np.random.default_rng(13)
    ic = np.sort(rng.choice(m.n_c, 512, replace=False))
    np.savez_compressed(OUT, member=np.array(MEMBER), steps=np.array(STEPS), dt=np.array(dt), idx_c=ic,
                        a_c_norm=np.array([np.linalg.norm(a) for a in tr.a_c]),
                        a_c_sample=np.array([a[ic] for a in tr.a_c]), a_c_final=tr.a_c[-1],
                        iters_prev=np.array(tr.iters[O.FAM_PREV]), iters_cur=np.array(tr.iters[O.FAM_CUR]))
    print(f"wrote {OUT} in {time.time() - t0:.0f} s", flush=True)


if __name__ == "__main__":
    main()
