"""K1 finish-time spread of the TMA PCG kernel across CTAs (load imbalance).

Needs a -DMQ_TRACE_SPREAD build (tools/build_variant.py sp -DMQ_TRACE_SPREAD):
    MQ_LIB_PATH=variants/sp.so MQ_PCG_TRACE=1 MQ_PCG_KERNEL=brick [MQ_PCG_SYNC=1] python tools/k1_spread.py
Prints, for configs[2] and configs[4], the per-CTA %globaltimer at the end of
K1 of iteration 10 relative to the earliest CTA.
"""
import ctypes, sys, numpy as np
sys.path.insert(0, '/root/repo')
from paper_1611_06721_b200 import _lib, configs as C
from paper_1611_06721_b200._lib import check
from paper_1611_06721_b200.device import DeviceGrid
for cfg in (2, 4):
    prob = C.make_problem(cfg)
    g = DeviceGrid(prob)
    b, x = g.alloc(), g.alloc()
    g.upload(prob.pattern, b)
    rep = _lib.SolveReportC()
    for _ in range(2):
        check(g.lib.mq_pcg_solve_dev(g.ctx, ctypes.c_void_p(b), None, ctypes.c_void_p(x), 1e-8, 0.0, 20, 1, ctypes.byref(rep)), allow=(0, 1))
    st = np.zeros(2048, dtype=np.uint64)
    check(g.lib.mq_pcg_trace(g.ctx, st.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), 2048))
    name, grid = g.pcg_kernel()
    t = st[1024:1024 + grid].astype(np.float64)
    t = (t - t.min()) / 1e3
    print(cfg, name, grid, "K1-end spread us: min 0 median %.2f p90 %.2f max %.2f" % (np.median(t), np.percentile(t, 90), t.max()))
    sm = st[1536:1536 + grid].astype(np.int64)
    if sm.any():  # pcg_tma1_kernel also records %smid: CTAs alone on their SM vs sharing one
        cnt = np.bincount(sm)[sm]
        lone, shared = t[cnt == 1], t[cnt >= 2]
        print("   alone on an SM: %d CTAs, median %.2f max %.2f; sharing: %d CTAs, median %.2f max %.2f"
              % (lone.size, np.median(lone) if lone.size else -1, lone.max() if lone.size else -1,
                 shared.size, np.median(shared), shared.max()))
    else:  # by launch order: first 148 CTAs vs rest
        print("   first 148 CTAs median %.2f, last %d median %.2f" % (np.median(t[:148]), grid - 148, np.median(t[148:])))
    g.close()
