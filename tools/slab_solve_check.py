"""Fused slab PCG (emulated ranks) vs the single-context PCG on a config
grid, with and without a start vector (diagnostic).

    python tools/slab_solve_check.py --config 4 --world 2
"""
import argparse
import ctypes
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--world", type=int, default=2)
    ap.add_argument("--iters", type=int, default=5000)
    args = ap.parse_args()
    import numpy as np

    from paper_1611_06721_b200 import _lib, configs as C
    from paper_1611_06721_b200._lib import check, dptr
    from paper_1611_06721_b200.device import DeviceGrid
    from paper_1611_06721_b200.slab import SlabGrid, fused_slab_pcg_solve_local
    from paper_1611_06721_b200.slabstep import global_compact_index
    prob = C.make_problem(args.config)
    g = DeviceGrid(prob)
    n = g.n_n
    gidx = global_compact_index(prob.material)
    slabs = [SlabGrid(prob, r, args.world) for r in range(args.world)]
    idx = [gidx[s.partition()] for s in slabs]
    rng = np.random.default_rng(3)
    b = np.asarray(prob.pattern, np.float64)
    out = {}
    for label, x0 in (("zero", None), ("start", rng.standard_normal(n) * 1e-9)):
        xs = np.empty(n)
        rep = _lib.SolveReportC()
        check(g.lib.mq_pcg_solve_host(g.ctx, dptr(b), dptr(x0) if x0 is not None else None, dptr(xs), 1e-8, 0.0,
                                      args.iters, 1, ctypes.byref(rep)), allow=(0, 1))
        for s, ix in zip(slabs, idx):
            s.upload(b[ix], s.b)
            s.upload(x0[ix] if x0 is not None else np.zeros(ix.size), s.x)
        it, relres, conv, app = fused_slab_pcg_solve_local(slabs, x0_given=x0 is not None, rel_tol=1e-8,
                                                           max_iter=args.iters)
        x = np.zeros(n)
        for s, ix in zip(slabs, idx):
            x[ix] = s.download(s.x)
        out[label] = {"single_iters": rep.iterations, "slab_iters": it, "slab_rel": relres,
                      "x_rel": float(np.linalg.norm(x - xs) / np.linalg.norm(xs))}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
