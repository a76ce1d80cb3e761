"""Host-API step breakdown (explicit_euler_step + recover_an + probe_b).

    python tools/e2e_breakdown.py [--steps 10]
"""
import argparse
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    args = ap.parse_args()
    from paper_1611_06721_b200 import PcgConfig, SchurOperator, configs as C
    from paper_1611_06721_b200.schur import explicit_euler_step, recover_an
    spec = C.config_spec(1)
    op = SchurOperator(C.make_problem(1), pcg=PcgConfig(rel_tol=1e-8), strategy="cspe", max_cols=5)
    op.set_probe()
    a, t = np.zeros(op.grid.n_c), 0.0
    recover_an(op, a, t)
    for s in range(3):
        a, _ = explicit_euler_step((a, t), spec.dt, op, s + 1)
        t += spec.dt
        recover_an(op, a, t)
    tm = {"euler": 0.0, "recover": 0.0, "probe": 0.0}
    for s in range(args.steps):
        t0 = time.perf_counter()
        a, _ = explicit_euler_step((a, t), spec.dt, op, s + 4)
        t1 = time.perf_counter()
        t += spec.dt
        recover_an(op, a, t)
        t2 = time.perf_counter()
        op.probe_b()
        t3 = time.perf_counter()
        tm["euler"] += t1 - t0
        tm["recover"] += t2 - t1
        tm["probe"] += t3 - t2
    n = args.steps
    print("ms per step: " + "  ".join(f"{k} {1000 * v / n:.3f}" for k, v in tm.items()),
          f" total {1000 * sum(tm.values()) / n:.3f}")
    # raw copies
    x = np.zeros(op.grid.n_n)
    d = op.grid.alloc()
    t0 = time.perf_counter()
    for _ in range(n):
        op.grid.upload(x, d)
    t1 = time.perf_counter()
    for _ in range(n):
        op.grid.download(d)
    t2 = time.perf_counter()
    print(f"n_n vector ({8 * op.grid.n_n / 1e6:.1f} MB): upload {1000 * (t1 - t0) / n:.3f} ms, "
          f"download {1000 * (t2 - t1) / n:.3f} ms")


if __name__ == "__main__":
    main()
