"""Concurrent ensemble members on one GPU (configs[3] exploration).

    python tools/ensemble_concurrency.py --members 4 --budget 37 --steps 10

Each member gets its own context/stream; its PCG kernel runs on a slice of
`budget` SMs; steps of all members are enqueued interleaved (CUDA graphs)
and member-steps/s is taken over the whole group.
"""
import argparse
import ctypes
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--members", type=int, default=4)
    ap.add_argument("--budget", type=int, default=0)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()
    from paper_1611_06721_b200 import PcgConfig, SchurOperator, _lib
    from paper_1611_06721_b200 import configs as C
    from paper_1611_06721_b200._lib import check, dptr
    from paper_1611_06721_b200.ensemble import member_problem
    from paper_1611_06721_b200.schur import recover_an
    spec = C.config_spec(3)
    ops = []
    n = args.warmup + args.steps
    for m in range(args.members):
        prob, jf, kf, dt = member_problem(m)
        op = SchurOperator(prob, pcg=PcgConfig(rel_tol=1e-8), strategy="cspe", max_cols=5)
        check(op.lib.mq_ctx_set_sm_budget(op.grid.ctx, args.budget))
        op.set_probe()
        recover_an(op, np.zeros(op.grid.n_c), 0.0)
        op._set_state(np.zeros(op.grid.n_c), 0.0)
        tt = [0.0]
        for _ in range(n):
            tt.append(tt[-1] + dt)
        wave = np.array([float(prob.waveform(t)) for t in tt])
        dts = np.full(n, dt)
        check(op.lib.mq_run_prepare(op.grid.ctx, n, dptr(dts), dptr(wave), 1))
        ops.append(op)
    lib = ops[0].lib
    for op in ops:
        check(lib.mq_run_steps(op.grid.ctx, args.warmup, 1, None))
    for op in ops:
        op.grid.sync()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        for op in ops:
            check(lib.mq_run_steps(op.grid.ctx, 1, 1, None))
    for op in ops:
        op.grid.sync()
    el = time.perf_counter() - t0
    its = []
    for op in ops:
        it = np.zeros((n, 4), dtype=np.int32)
        failed = ctypes.c_int64()
        check(lib.mq_run_finish(op.grid.ctx, _lib.i32ptr(it), ctypes.byref(failed)))
        its.append(int(it[args.warmup:].sum()))
    print(f"members={args.members} budget={args.budget} steps={args.steps}: "
          f"{args.members * args.steps / el:.1f} member-steps/s ({1000 * el / args.steps:.2f} ms per "
          f"group step), iterations per member {its}")


if __name__ == "__main__":
    main()
