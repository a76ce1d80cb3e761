"""Fused slab PCG (csrc/slab_fused.cu), ranks emulated as CTA groups on one GPU.

    python tools/slab_fused_bench.py --config 2 --ranks 1 2 4 8 --iters 200

Per rank count: one capped solve of the source pattern, us per iteration and
the 72 B/dof convention's GB/s (wall clock around the synchronous call).
"""
import argparse
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--ranks", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--iters", type=int, default=200)
    args = ap.parse_args()
    from paper_1611_06721_b200 import configs as C
    from paper_1611_06721_b200.device import DeviceGrid
    from paper_1611_06721_b200.slab import SlabGrid, fused_slab_pcg_solve_local
    prob = C.make_problem(args.config)
    with DeviceGrid(prob) as g:
        nc_all = g.partition()[0]
    for R in args.ranks:
        slabs = [SlabGrid(prob, r, R) for r in range(R)]
        idx = [np.searchsorted(nc_all, s.partition()) for s in slabs]
        for s, ix in zip(slabs, idx):
            s.upload(prob.pattern[ix], s.b)
        fused_slab_pcg_solve_local(slabs, x0_given=False, rel_tol=1e-8, max_iter=5)
        best = None
        for _ in range(2):
            t0 = time.perf_counter()
            it, rel, conv, app = fused_slab_pcg_solve_local(slabs, x0_given=False, rel_tol=1e-8,
                                                            max_iter=args.iters)
            el = time.perf_counter() - t0
            best = el if best is None else min(best, el)
        us = 1e6 * best / max(it, 1)
        gbs = 72.0 * nc_all.size / (us * 1e-6) / 1e9
        print(f"config {args.config} ranks {R}: {it} it, {us:.1f} us/it, {gbs:.0f} GB/s (72 B/dof/it)", flush=True)
        for s in slabs:
            s.close()


if __name__ == "__main__":
    main()
