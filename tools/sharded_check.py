"""Sharded step vs the single-context loop on one config grid (diagnostic).

    python tools/sharded_check.py --config 4 --world 2 --steps 1
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--world", type=int, default=2)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--strategy", default="cspe")
    args = ap.parse_args()
    import numpy as np

    from paper_1611_06721_b200 import PcgConfig, configs as C, run_explicit
    from paper_1611_06721_b200.slabstep import run_explicit_sharded
    spec = C.config_spec(args.config)
    prob = C.make_problem(args.config)
    n = args.steps
    one = run_explicit(prob, t_end=n * spec.dt, dt=spec.dt, strategy=args.strategy, pcg=PcgConfig(rel_tol=1e-8),
                       max_cols=5, output_period=spec.dt * (1 - 1e-3), record_states=True)
    res = run_explicit_sharded(prob, n, spec.dt, world=args.world, strategy=args.strategy, max_cols=5,
                               record_states=True)

    def rel(a, b):
        return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
    out = {"config": args.config, "world": args.world,
           "iters_single": one.step_iterations.tolist(), "iters_sharded": res.step_iterations.tolist(),
           "a_c_rel": [rel(res.a_c_history[i], one.a_c_history[i]) for i in range(n)],
           "a_n_rel": [rel(res.a_n_history[i], one.a_n_history[i]) for i in range(n)],
           "a_n_norms": [float(np.linalg.norm(res.a_n_history[i])) for i in range(n)],
           "a_n_norms_single": [float(np.linalg.norm(one.a_n_history[i])) for i in range(n)]}
    d = res.a_n_history[0] - one.a_n_history[0]
    idx = np.argsort(-np.abs(d))[:5]
    out["worst_a_n_idx"] = idx.tolist()
    out["worst_a_n"] = [[float(res.a_n_history[0][q]), float(one.a_n_history[0][q])] for q in idx]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
