"""Run a BASELINE config on one GPU: device CFL estimate (when the config has
no dt), then N explicit-Euler steps with recovery every step.

    python tools/run_config.py --config 4 --steps 5
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    args = ap.parse_args()
    import numpy as np

    from paper_1611_06721_b200 import PcgConfig, SchurOperator, estimate_cfl, run_explicit
    from paper_1611_06721_b200 import configs as C
    spec = C.config_spec(args.config)
    t0 = time.time()
    prob = C.make_problem(args.config)
    op = SchurOperator(prob, pcg=PcgConfig(rel_tol=spec.rel_tol, max_iter=spec.max_iter),
                       strategy=spec.strategy, max_cols=spec.max_cols, n_pod=spec.n_pod)
    setup = time.time() - t0
    out = {"config": spec.name, "n_n": op.grid.n_n, "n_c": op.grid.n_c, "setup_s": setup}
    dt = spec.dt
    if dt is None:
        t1 = time.time()
        est = estimate_cfl(op)
        dt = est.dt_max
        out.update(cfl_lambda=est.lambda_max, cfl_dt=dt, cfl_power_iters=est.power_iters,
                   cfl_s=time.time() - t1)
    n = args.warmup + args.steps
    t2 = time.time()
    res = run_explicit(prob, t_end=n * dt, dt=dt, output_period=dt * (1 - 1e-3), op=op)
    wall = time.time() - t2
    it = res.step_iterations
    out.update(dt=dt, steps=n, wall_s=wall, steps_per_s=n / wall,
               iterations_per_step=it.sum(axis=1).tolist(),
               final_a_c_norm=float(np.linalg.norm(res.final_a_c)),
               aggregates={k: v for k, v in res.aggregates.items() if k != "wall_seconds"})
    print(json.dumps(out))


if __name__ == "__main__":
    main()
