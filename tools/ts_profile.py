"""Profiling driver for the tall-skinny start-vector kernels (CSPE / POD):
N explicit-Euler steps (recovery every step) of a BASELINE config's grid with
the chosen strategy, so that an ncu pass filtered on the k_mdot /
k_axpy_dots / k_comb / k_cspe_product / k_pod_* kernels sees them at size.

    python tools/ts_profile.py --config 2 --strategy cspe --steps 6
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--strategy", default=None)
    ap.add_argument("--steps", type=int, default=6)
    args = ap.parse_args()
    import numpy as np

    from paper_1611_06721_b200 import PcgConfig, SchurOperator, run_explicit
    from paper_1611_06721_b200 import configs as C
    spec = C.config_spec(args.config)
    prob = C.make_problem(args.config)
    strategy = args.strategy or spec.strategy
    op = SchurOperator(prob, pcg=PcgConfig(rel_tol=spec.rel_tol, max_iter=spec.max_iter),
                       strategy=strategy, max_cols=spec.max_cols,
                       n_pod=spec.n_pod)
    dt = spec.dt
    res = run_explicit(prob, t_end=args.steps * dt, dt=dt, output_period=dt * (1 - 1e-3), op=op)
    print(json.dumps({"config": spec.name, "strategy": strategy, "n_n": op.grid.n_n,
                      "iterations": res.step_iterations.tolist(),
                      "final_a_c_norm": float(np.linalg.norm(res.final_a_c))}))


if __name__ == "__main__":
    main()
