"""Every BASELINE config at its full length on one GPU (device-resident loop,
recovery and the B probe every step): completes without a step failure, and
a summary per run — steps/s, iterations per family, final field norms, start
vector diagnostics — as JSON lines (profiles/r0N_full_runs.jsonl).

    python tools/full_runs.py [--only 0,1,2,3,4]

configs[3]: members 0, 1 and 255 of the 256-member ensemble (the others are
the same computation with other J/kappa factors); configs[1] with both of its
start-vector strategies.
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def summary(name, res, wall, steps, extra=None):
    it = np.asarray(res.step_iterations)
    fam = ["source", "coupling_previous", "source_recovery", "coupling_current"]
    out = {"run": name, "steps": steps, "wall_s": round(wall, 3), "steps_per_s": round(steps / wall, 2),
           "pcg_iterations_total": int(it.sum()),
           "iterations": {f: {"min": int(it[:, q].min()), "mean": round(float(it[:, q].mean()), 1),
                              "max": int(it[:, q].max())} for q, f in enumerate(fam)},
           "final_a_c_norm": float(np.linalg.norm(res.final_a_c)),
           "final_a_n_norm": float(np.linalg.norm(res.final_a_n)) if res.final_a_n is not None else None,
           "probe_b_last": float(res.probe_b[-1]) if len(res.probe_b) else None,
           "basis_cols_last": int(res.basis_cols[-1]) if len(res.basis_cols) else None,
           "pod_k_last": int(res.pod_k[-1]) if len(res.pod_k) else None,
           "aggregates": {k: v for k, v in res.aggregates.items() if k != "wall_seconds"}}
    out.update(extra or {})
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="0,1,2,3,4")
    args = ap.parse_args()
    only = {int(x) for x in args.only.split(",")}
    from paper_1611_06721_b200 import PcgConfig, run_explicit
    from paper_1611_06721_b200 import configs as C
    from paper_1611_06721_b200 import ensemble as E
    runs = []
    for idx in (0, 1, 2, 4):
        if idx not in only:
            continue
        spec = C.config_spec(idx)
        strategies = ["cspe", "pod"] if idx == 1 else [spec.strategy]
        for strat in strategies:
            prob = C.make_problem(idx)
            t0 = time.time()
            res = run_explicit(prob, t_end=spec.steps * spec.dt, dt=spec.dt, strategy=strat,
                               pcg=PcgConfig(rel_tol=spec.rel_tol, max_iter=spec.max_iter),
                               max_cols=spec.max_cols, n_pod=spec.n_pod,
                               output_period=spec.dt * (1 - 1e-3), probe="device")
            wall = time.time() - t0
            runs.append(summary(f"{spec.name}_{strat}", res, wall, spec.steps,
                                {"dt": spec.dt, "n_pod": spec.n_pod if strat == "pod" else None}))
            print(json.dumps(runs[-1]), flush=True)
    if 3 in only:
        spec = C.config_spec(3)
        for member in (0, 1, 255):
            prob, jf, kf, dt = E.member_problem(member)
            t0 = time.time()
            res = run_explicit(prob, t_end=spec.steps * dt, dt=dt, strategy="cspe",
                               pcg=PcgConfig(rel_tol=1e-8, max_iter=5000), max_cols=5,
                               output_period=dt * (1 - 1e-3), probe="device")
            wall = time.time() - t0
            runs.append(summary(f"cfg3_member{member}", res, wall, spec.steps,
                                {"dt": dt, "j_factor": jf, "kappa_factor": kf}))
            print(json.dumps(runs[-1]), flush=True)


if __name__ == "__main__":
    main()
