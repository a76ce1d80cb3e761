"""Determinism check of the device loop: the same configs[0] POD run twice
eager and twice as graph replays must give bit-identical states and
iteration counts.

    python tools/det_check.py
"""
import numpy as np, sys
sys.path.insert(0, '/root/repo')
from paper_1611_06721_b200 import configs as C, PcgConfig, run_explicit
spec = C.config_spec(0)
outs = []
for g in (False, False, True, True):
    r = run_explicit(C.make_problem(0), t_end=30 * spec.dt, dt=spec.dt, strategy="pod", pcg=PcgConfig(rel_tol=1e-8),
                     output_period=spec.dt * (1 - 1e-3), n_pod=20, eps_pod=1e-4, use_graph=g)
    outs.append(r)
for i in range(1, 4):
    print(i, np.array_equal(outs[0].final_a_c, outs[i].final_a_c), np.abs(outs[0].final_a_c - outs[i].final_a_c).max(),
          np.array_equal(outs[0].step_iterations, outs[i].step_iterations))
