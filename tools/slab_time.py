"""Per-iteration time of the fused slab PCG kernel on one GPU's share of a
multi-GPU configs[4] run (diagnostic): rank 0's slab of a WORLD-way split of
the 256^3 grid, solved alone (its neighbours' ghost planes stay zero), a fixed
iteration budget, CUDA-synchronised host clock.

    MQ_PCG_SYNC=1|2 python tools/slab_time.py --world 4 --iters 60
"""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--world", type=int, default=4)
    ap.add_argument("--iters", type=int, default=60)
    args = ap.parse_args()
    import numpy as np

    from paper_1611_06721_b200 import configs as C
    from paper_1611_06721_b200.slab import SlabGrid, fused_slab_pcg_solve_local
    s = SlabGrid(C.make_problem(args.config), 0, args.world)
    n = s.partition().size
    b = np.random.default_rng(5).standard_normal(n)
    s.upload(b, s.b)
    best = None
    for _ in range(3):
        s.upload(np.zeros(n), s.x)
        t0 = time.perf_counter()
        it, rel, conv, app = fused_slab_pcg_solve_local([s], x0_given=False, rel_tol=1e-30, max_iter=args.iters)
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    print(f"config {args.config} world {args.world} slab planes {s.n_planes} n_own {n} iters {it} "
          f"{1e6 * best / it:.1f} us/it (launch incl. init, best of 3)")
    s.close()


if __name__ == "__main__":
    main()
