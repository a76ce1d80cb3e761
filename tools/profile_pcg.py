"""Profiling driver: one fused-PCG solve on a BASELINE config grid.

    python tools/profile_pcg.py --config 2 --iters 20 [--kernel brick|simple]

Runs a warm-up solve, then one solve capped at --iters iterations (so an ncu
replay stays short), and prints the CUDA-event time per iteration.
"""
import argparse
import ctypes
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--kernel", default=os.environ.get("MQ_PCG_KERNEL", ""))
    ap.add_argument("--spmv", action="store_true", help="also time K_n SpMV launches")
    ap.add_argument("--zero", action="store_true", help="also time zero-iteration solves")
    args = ap.parse_args()
    if args.kernel:
        os.environ["MQ_PCG_KERNEL"] = args.kernel
    from paper_1611_06721_b200 import _lib, configs as C
    from paper_1611_06721_b200._lib import check
    from paper_1611_06721_b200.device import DeviceGrid
    prob = C.make_problem(args.config)
    g = DeviceGrid(prob)
    lib = g.lib
    b, x = g.alloc(), g.alloc()
    g.upload(prob.pattern, b)
    rep = _lib.SolveReportC()
    rc = lib.mq_pcg_solve_dev(g.ctx, ctypes.c_void_p(b), None, ctypes.c_void_p(x), 1e-8, 0.0,
                              args.iters, 1, ctypes.byref(rep))
    check(rc, allow=(0, 1))
    check(lib.mq_pcg_stats(g.ctx, None, None, None, 1))
    rc = lib.mq_pcg_solve_dev(g.ctx, ctypes.c_void_p(b), None, ctypes.c_void_p(x), 1e-8, 0.0,
                              args.iters, 1, ctypes.byref(rep))
    check(rc, allow=(0, 1))
    ms, it = ctypes.c_double(), ctypes.c_int64()
    check(lib.mq_pcg_stats(g.ctx, ctypes.byref(ms), ctypes.byref(it), None, 0))
    n = g.n_n
    gbs = 72.0 * n * rep.iterations / (ms.value * 1e-3) / 1e9
    print(f"config {args.config} kernel={args.kernel} n_n={n} iters={rep.iterations} "
          f"time={ms.value:.3f} ms  {1000*ms.value/max(rep.iterations,1):.1f} us/it  "
          f"{gbs:.0f} GB/s (72 B/dof/it)")
    if os.environ.get("MQ_PCG_TRACE"):
        import numpy as np
        st = np.zeros(4 * 64 + 1, dtype=np.uint64)
        check(lib.mq_pcg_trace(g.ctx, st.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), st.size))
        n = min(64, rep.iterations)
        s = st[1:4 * n + 1].reshape(n, 4).astype(np.float64)
        prev = np.concatenate([[float(st[0])], s[:-1, 3]])
        k1, b1, k2, b2 = s[:, 0] - prev, s[:, 1] - s[:, 0], s[:, 2] - s[:, 1], s[:, 3] - s[:, 2]
        print(f"  per-iteration us (CTA 0, iterations 2..{n}): K1 {k1[1:].mean()/1e3:.2f}  barrier1 "
              f"{b1[1:].mean()/1e3:.2f}  K2 {k2[1:].mean()/1e3:.2f}  barrier2 {b2[1:].mean()/1e3:.2f}  "
              f"(init {k1[0]/1e3:.2f})")
    if os.environ.get("MQ_TRACE_MARCH"):
        # pcg_tma_kernel built with -DMQ_TRACE_MARCH: CTA 0, iteration 10, per
        # plane step i: [before TMA wait of plane i+1, after it, after the
        # convert, after the __syncthreads]; the stencil of plane i follows
        import numpy as np
        st = np.zeros(1300 + 140, dtype=np.uint64)
        check(lib.mq_pcg_trace(g.ctx, st.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), st.size))
        m = st[1300:1300 + 4 * 31].reshape(31, 4).astype(np.float64)
        wait = m[:, 1] - m[:, 0]
        conv = m[:, 2] - m[:, 1]
        sync = m[:, 3] - m[:, 2]
        sten = m[1:, 0] - m[:-1, 3]
        print(f"  march us per plane step (CTA 0): TMA wait {wait[2:].mean()/1e3:.3f}  convert {conv[2:].mean()/1e3:.3f}  "
              f"syncthreads {sync[2:].mean()/1e3:.3f}  stencil+prefetch {sten[2:].mean()/1e3:.3f}  "
              f"step {np.diff(m[:, 0])[2:].mean()/1e3:.3f}")
        e = st[1300 + 128:1300 + 132].astype(np.float64)
        print(f"  march entry -> plane i0-1 converted {(e[1]-e[0])/1e3:.2f} us, -> prologue done "
              f"{(e[2]-e[0])/1e3:.2f} us, march total {(e[3]-e[0])/1e3:.2f} us")
        print("  first steps (us): wait " + " ".join(f"{v/1e3:.2f}" for v in wait[:6]) +
              " | step " + " ".join(f"{v/1e3:.2f}" for v in np.diff(m[:, 0])[:6]))
    if os.environ.get("MQ_TRACE_FINE") and g.pcg_kernel()[0].startswith("pcg_resident1"):
        # single-reduction kernel: fine stamps 0..3 = loop top, stencil + dots
        # + Ap stores done, partial sums read, own + halo update done;
        # coarse 1/2 = before / after the barrier
        import numpy as np
        st = np.zeros(1024, dtype=np.uint64)
        check(lib.mq_pcg_trace(g.ctx, st.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), st.size))
        coarse = st[1:4 * 33 + 1].reshape(33, 4).astype(np.float64)
        fine = st[320:320 + 8 * 32].reshape(32, 8).astype(np.float64)
        rows = []
        for it in range(2, 31):
            f, c = fine[it], coarse[it]
            rows.append([f[1] - f[0], c[0] - f[1], c[1] - c[0], f[2] - c[1], f[3] - f[2], fine[it + 1][0] - f[3]])
        r = np.mean(np.array(rows), axis=0) / 1e3
        names = ["sync_stencil_dots", "bsum_pstore", "barrier", "psum", "update_own_halo", "tail"]
        print("  fine us: " + "  ".join(f"{n} {v:.2f}" for n, v in zip(names, r)) + f"  total {r.sum():.2f}")
    elif os.environ.get("MQ_TRACE_FINE"):
        import numpy as np
        st = np.zeros(1024, dtype=np.uint64)
        check(lib.mq_pcg_trace(g.ctx, st.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), st.size))
        coarse = st[1:4 * 33 + 1].reshape(33, 4).astype(np.float64)
        fine = st[320:320 + 8 * 32].reshape(32, 8).astype(np.float64)
        rows = []
        for it in range(2, 32):   # iteration it+1 (1-based), skip the first
            f = fine[it]
            b1s, b1e, k2e, b2e = coarse[it]  # stamps 1..4 of this iteration
            rows.append([f[1] - f[0], f[2] - f[1], f[3] - f[2], f[4] - f[3], f[5] - f[4],
                         b1s - f[5], b1e - b1s, f[6] - b1e, f[7] - f[6], k2e - f[7], b2e - k2e,
                         fine[it + 1][0] - b2e if it + 1 < 32 else np.nan])
        r = np.nanmean(np.array(rows), axis=0) / 1e3
        names = ["own_p", "halo", "sync", "stencil", "bsum1", "pstore", "bar1", "psum1", "k2loop",
                 "bsum2", "bar2", "psum2"]
        print("  fine us: " + "  ".join(f"{n} {v:.2f}" for n, v in zip(names, r)))
    if args.zero:
        # launch cost of a solve that converges at its initial residual (the
        # SOURCE-family solves of every step): x0 = the solution just found
        check(lib.mq_pcg_stats(g.ctx, None, None, None, 1))
        for _ in range(20):
            rc = lib.mq_pcg_solve_dev(g.ctx, ctypes.c_void_p(b), ctypes.c_void_p(x), ctypes.c_void_p(x), 1e-6,
                                      0.0, 10, 1, ctypes.byref(rep))
            check(rc, allow=(0, 1))
        ms0, it0 = ctypes.c_double(), ctypes.c_int64()
        check(lib.mq_pcg_stats(g.ctx, ctypes.byref(ms0), ctypes.byref(it0), None, 0))
        ms = ms0
        print(f"  zero-iteration solve (x0 exact, iters={rep.iterations}): {1000 * ms.value / 20:.1f} us per launch")
        if os.environ.get("MQ_TRACE_FINE") and os.environ.get("MQ_PCG_TRACE"):
            import numpy as np
            st = np.zeros(320, dtype=np.uint64)
            check(lib.mq_pcg_trace(g.ctx, st.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), st.size))
            t = st[[0, 301, 302, 303, 304, 305, 306]].astype(np.float64)
            d = np.diff(t) / 1e3
            names = ["residual", "bsum_pstore", "barrier", "psum", "halo_r", "tail"]
            print("  init us (CTA 0, last launch): " + "  ".join(f"{n} {v:.2f}" for n, v in zip(names, d)))
    if args.spmv:
        y = g.alloc()
        lib.mq_timer_start(g.ctx)
        for _ in range(20):
            check(lib.mq_kn_apply_dev(g.ctx, ctypes.c_void_p(b), ctypes.c_void_p(y)))
        t = ctypes.c_double()
        lib.mq_timer_stop(g.ctx, ctypes.byref(t))
        print(f"kn_apply: {1000*t.value/20:.1f} us  ({16.0*n/(t.value/20*1e-3)/1e9:.0f} GB/s at 16 B/dof)")
    g.close()


if __name__ == "__main__":
    main()
