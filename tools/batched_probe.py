"""Member-batched PCG vs one member at a time at 64^3 (configs[1]/[3] grid):
device time per member-iteration of mq_pcg_solve_batched_host for nb = 1, 2,
4, 8 against the shared-memory-resident single-member kernel.

    python tools/batched_probe.py
"""
import ctypes
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import numpy as np

    from paper_1611_06721_b200 import _lib, configs as C
    from paper_1611_06721_b200._lib import check
    from paper_1611_06721_b200.device import DeviceGrid
    g = DeviceGrid(C.make_problem(1))
    rng = np.random.default_rng(0)
    rhs = [g.kn_apply(rng.standard_normal(g.n_n)) for _ in range(8)]
    out = {"grid": "64^3", "n_n": g.n_n}
    # single member, resident kernel, device vectors
    b, x = g.alloc(), g.alloc()
    g.upload(rhs[0], b)
    rep = _lib.SolveReportC()
    check(g.lib.mq_pcg_solve_dev(g.ctx, ctypes.c_void_p(b), None, ctypes.c_void_p(x), 1e-8, 0.0, 5000, 1,
                                 ctypes.byref(rep)))
    check(g.lib.mq_pcg_stats(g.ctx, None, None, None, 1))
    check(g.lib.mq_pcg_solve_dev(g.ctx, ctypes.c_void_p(b), None, ctypes.c_void_p(x), 1e-8, 0.0, 5000, 1,
                                 ctypes.byref(rep)))
    ms, it = ctypes.c_double(), ctypes.c_int64()
    check(g.lib.mq_pcg_stats(g.ctx, ctypes.byref(ms), ctypes.byref(it), None, 0))
    out["single"] = {"kernel": g.pcg_kernel()[0], "iterations": rep.iterations,
                     "us_per_member_iteration": 1000.0 * ms.value / rep.iterations}
    for nb in (1, 2, 4, 8):
        bm = np.stack(rhs[:nb])
        g.pcg_batched(bm, None, rel_tol=1e-8)  # warm-up
        _, reps, kms = g.pcg_batched(bm, None, rel_tol=1e-8)
        iters = [r[0] for r in reps]
        out[f"batched_{nb}"] = {"iterations": iters, "launch_ms": kms,
                               "us_per_iteration": 1000.0 * kms / max(iters),
                               "us_per_member_iteration": 1000.0 * kms / sum(iters)}
    g.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
