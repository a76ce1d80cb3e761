"""Sharded explicit-Euler step over i-slabs (BASELINE configs[4]).

The SchurOperator step of the reference (``mq/schur.py:379-405``
``explicit_euler_step``, ``408-419`` ``recover_an``) with the CSPE start
vectors (``mq/startvec.py:158-225``) on a grid whose K_n-sized vectors are
split into i-slabs, one slab per rank (``slab.py``).  Per step:

    source rhs (own rows)          -> project (all-reduce k) -> fused slab PCG
                                   -> insert (all-reduces k+1, k+1, 1, k'+1;
                                      one halo exchange before K u)
    K_cn^T a_c (own rows)          -> the same for the coupling family
    y_cpl - y_src (halo exchange)  -> Brauer nu + Euler on the owned conducting
                                      edges -> all-gather -> a_c on every rank
    recovery: the same two solves at the new state (families SOURCE and
    COUPLING_CURRENT), a_n = y_src - y_cur on each slab.

The device side is ``csrc/solver_slab.cuh`` (C ABI ``mq_ss_*``): the
single-device tall-skinny kernels and CSPE decision code run on each slab;
every reduction leaves a rank partial that the communicator sums over the
ranks in rank order, so all ranks take identical decisions.  The PCG solves
are the fused slab kernel (``csrc/slab_fused.cu``): one persistent kernel per
rank with the halo stores and the rank all-reduce inside it.

Communicators (``slab.py``): ``LoopbackComm`` — every slab in this process
(the single-GPU emulation; the PCG then runs all slabs as the CTA groups of
one cooperative launch), ``TorchComm`` — one slab per process over
torch.distributed (NCCL between GPUs, gloo on CPU), with the fused PCG over
CUDA-IPC-mapped neighbour buffers.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import check, dptr
from .configs import noncond_positions
from .krylov import IndefiniteOperatorError
from .schur import StepFailureError
from .slab import LoopbackComm, SlabGrid, TorchComm, _DevArray, fused_peer_setup

__all__ = ["SlabStepGrid", "SlabStepper", "ShardedRun", "run_explicit_sharded", "global_compact_index"]

NPART = 34  # MQ_SS_NPART
_VEC = {"rhs_src": 0, "rhs_cpl": 1, "y_src": 2, "y_cpl": 3, "y_cur": 4, "w2": 5, "dvec": 6}
FAM_SOURCE, FAM_CUR, FAM_PREV = _lib.FAM_SOURCE, _lib.FAM_COUPLING_CURRENT, _lib.FAM_COUPLING_PREVIOUS


def global_compact_index(material: np.ndarray) -> np.ndarray:
    """Global edge id -> compact K_n index (-1 off the partition), the
    reference's numbering (model.py:455-464)."""
    return noncond_positions(material)[1]


class SlabStepGrid(SlabGrid):
    """One slab with the sharded-step state (``mq_ss_init``)."""

    def __init__(self, problem, rank: int, world: int, device: int = 0, *, cfg: _lib.SolverCfg,
                 gidx_all: np.ndarray | None = None):
        super().__init__(problem, rank, world, device)
        gidx_all = global_compact_index(problem.material) if gidx_all is None else gidx_all
        self.gidx = gidx_all[self.partition()]  # compact global index of every own dof
        if (self.gidx < 0).any():
            raise RuntimeError("slab partition disagrees with the global numbering")
        pattern = np.ascontiguousarray(np.asarray(problem.pattern, np.float64)[self.gidx])
        check(self.lib.mq_ss_init(self.ctx, ctypes.byref(cfg), dptr(pattern)))
        info = np.zeros(4, dtype=np.int64)
        check(self.lib.mq_ss_info(self.ctx, _lib.i64ptr(info)))
        self.n_c, self.n_own = int(info[0]), int(info[1])
        self.owned = np.zeros(self.n_own, dtype=np.int64)
        if self.n_own:
            check(self.lib.mq_ss_owned(self.ctx, _lib.i64ptr(self.owned)))
        self.vecs = {}
        for name, w in _VEC.items():
            p = ctypes.c_void_p()
            check(self.lib.mq_ss_vec(self.ctx, w, ctypes.byref(p)))
            self.vecs[name] = p.value

    def _ptr(self, name):
        return self.vecs[name] if name in self.vecs else super()._ptr(name)

    # -- phases (csrc/solver_slab.cuh) ----------------------------------------
    def state_set(self, a_c):
        check(self.lib.mq_ss_state_set(self.ctx, dptr(np.ascontiguousarray(a_c, np.float64))))

    def state_get(self) -> np.ndarray:
        out = np.empty(self.n_c)
        check(self.lib.mq_ss_state_get(self.ctx, dptr(out)))
        return out

    def rhs(self, which: int, wave: float = 0.0):
        check(self.lib.mq_ss_rhs(self.ctx, int(which), float(wave)))

    def project(self, fam: int, which: int) -> np.ndarray:
        part = np.zeros(NPART)
        check(self.lib.mq_ss_project(self.ctx, int(fam), int(which), dptr(part)))
        return part

    def start(self, fam: int, tot: np.ndarray):
        check(self.lib.mq_ss_start(self.ctx, int(fam), dptr(np.ascontiguousarray(tot)), ctypes.c_void_p(self.x)))

    def store(self, fam: int, rep: _lib.SolveReportC):
        check(self.lib.mq_ss_store(self.ctx, int(fam), ctypes.c_void_p(self.x), ctypes.byref(rep)))

    def observe(self, fam: int, phase: int, tot=None):
        part = np.zeros(NPART)
        flag = ctypes.c_int32(0)
        t = dptr(np.ascontiguousarray(tot)) if tot is not None else None
        check(self.lib.mq_ss_observe(self.ctx, int(fam), int(phase), t, dptr(part), ctypes.byref(flag)))
        return part, int(flag.value)

    def euler_prep(self):
        check(self.lib.mq_ss_euler_prep(self.ctx))

    def euler(self, dt: float) -> np.ndarray:
        out = np.zeros(max(1, self.n_own))
        # a non-finite value is reported after the all-gather, on every rank
        check(self.lib.mq_ss_euler(self.ctx, float(dt), dptr(out)), allow=(0, _lib.MQ_NONFINITE))
        return out[: self.n_own]

    def a_n_local(self) -> np.ndarray:
        out = np.empty(self.n_n)
        check(self.lib.mq_ss_an(self.ctx, dptr(out)))
        return out

    def diagnostics(self) -> _lib.Diag:
        d = _lib.Diag()
        check(self.lib.mq_ss_diag(self.ctx, ctypes.byref(d)))
        return d

    def cspe_export(self, fam: int):
        """(U, K U) on this slab's own dofs (n_n x k each) and the Galerkin matrix."""
        k = ctypes.c_int32()
        U = np.empty((32, self.n_n))
        KU = np.empty((32, self.n_n))
        G = np.empty(32 * 32)
        check(self.lib.mq_ss_cspe_export(self.ctx, int(fam), ctypes.byref(k), dptr(U), dptr(KU), dptr(G)))
        kk = k.value
        return U[:kk].T.copy(), KU[:kk].T.copy(), G[:kk * kk].reshape(kk, kk).copy()

    def stage_b(self, which: str):
        """Copy the named rhs into this slab's PCG ``b`` (host-driven PCG)."""
        import torch
        n = self.total
        src = torch.as_tensor(_DevArray(self.vecs[which], n), device=f"cuda:{self.device}")
        dst = torch.as_tensor(_DevArray(self.b, n), device=f"cuda:{self.device}")
        self.sync()
        dst.copy_(src)
        torch.cuda.synchronize(self.device)


def _sum_rank_order(parts):
    tot = np.array(parts[0], dtype=np.float64, copy=True)
    for p in parts[1:]:
        tot = tot + p
    return tot


class _Loopback:
    """All slabs of the grid in this process (LoopbackComm semantics)."""

    def __init__(self):
        self.halo = LoopbackComm()

    def allreduce(self, parts):
        tot = _sum_rank_order(parts)
        return [tot for _ in parts]

    def allgather(self, arrays):
        return list(arrays)

    def exchange(self, slabs, names):
        self.halo.exchange(slabs, names)


class _Torch:
    """One slab per process over torch.distributed: partials all-gathered and
    summed in rank order (identical bits on every rank, whatever the
    backend's reduction tree), owned values all-gathered."""

    def __init__(self, dist, device=None):
        self.dist = dist
        self.halo = TorchComm(dist, device)
        # gloo moves host memory only
        self.device = "cpu" if (device is None or dist.get_backend() == "gloo") else device
        self.world = dist.get_world_size()

    def _gather(self, arr: np.ndarray) -> list[np.ndarray]:
        import torch
        n = np.array([arr.size], dtype=np.int64)
        sizes = [torch.zeros(1, dtype=torch.int64, device=self.device) for _ in range(self.world)]
        self.dist.all_gather(sizes, torch.as_tensor(n, device=self.device))
        sizes = [int(s.item()) for s in sizes]
        m = max(1, max(sizes))
        buf = torch.zeros(m, dtype=torch.float64, device=self.device)
        buf[: arr.size] = torch.as_tensor(arr, device=self.device)
        out = [torch.zeros(m, dtype=torch.float64, device=self.device) for _ in range(self.world)]
        self.dist.all_gather(out, buf)
        return [o[:s].cpu().numpy() for o, s in zip(out, sizes)]

    def allreduce(self, parts):
        (p,) = parts
        return [_sum_rank_order(self._gather(np.asarray(p, np.float64)))]

    def allgather(self, arrays):
        (a,) = arrays
        return self._gather(np.asarray(a, np.float64))

    def exchange(self, slabs, names):
        self.halo.exchange(slabs, names)


@dataclass
class ShardedRun:
    """run_explicit-like result of the sharded stepper."""

    step_iterations: np.ndarray            # (steps, 4): src, cpl_prev, src_rec, cpl_cur
    final_a_c: np.ndarray
    final_a_n: np.ndarray | None
    a_c_history: np.ndarray | None = None
    a_n_history: np.ndarray | None = None
    step_seconds: list = field(default_factory=list)
    aggregates: dict = field(default_factory=dict)


class SlabStepper:
    """explicit_euler_step / recover_an (schur.py:379-419) over i-slabs.

    ``ranks``: the slabs this process drives (all of them with the loopback
    communicator on one GPU; ``[rank]`` with ``dist``).  ``pcg``: "fused"
    (the fused slab kernel: one cooperative launch over the local slabs, or
    over IPC-mapped neighbours with ``dist``)."""

    def __init__(self, problem, world: int, *, dist=None, device: int = 0, strategy: str = "cspe",
                 max_cols: int = 5, rel_tol: float = 1e-8, abs_tol: float = 0.0, max_iter: int = 5000,
                 pcg: str = "fused", slabs=None, comm=None):
        if strategy not in ("zero", "previous", "cspe"):
            raise ValueError("the sharded step supports the zero / previous / cspe strategies")
        if pcg not in ("fused", "host"):
            raise ValueError("pcg must be 'fused' (one persistent kernel per rank) or 'host' (phase loop)")
        self.problem = problem
        self.world = int(world)
        self.strategy = strategy
        self.pcg_mode = pcg
        self.rel_tol, self.abs_tol, self.max_iter = float(rel_tol), float(abs_tol), int(max_iter)
        cfg = _lib.SolverCfg(_lib.STRAT[strategy], int(max_cols), 1, int(max_iter), 1e-4, float(rel_tol),
                             float(abs_tol), float(rel_tol))
        gidx_all = global_compact_index(problem.material)
        self.n_n = int((gidx_all >= 0).sum())
        self.dist = dist
        distributed = dist is not None and dist.is_initialized() and dist.get_world_size() > 1
        if distributed and dist.get_world_size() != self.world:
            raise ValueError("world size disagrees with torch.distributed")
        if comm is not None:
            self.comm = comm
        elif distributed:
            import torch
            dev = torch.device("cuda", device) if dist.get_backend() == "nccl" else None
            self.comm = _Torch(dist, dev)
        else:
            self.comm = _Loopback()
        if slabs is not None:
            # prebuilt slab objects with the SlabStepGrid phase methods (tests
            # drive numpy slabs through the same host sequence under gloo)
            self.slabs = list(slabs)
        else:
            ranks = [dist.get_rank()] if distributed else list(range(self.world))
            self.slabs = [SlabStepGrid(problem, r, self.world, device, cfg=cfg, gidx_all=gidx_all) for r in ranks]
        self.lib = getattr(self.slabs[0], "lib", None)
        self.n_c = self.slabs[0].n_c
        self.peer = pcg == "fused" and len(self.slabs) == 1 and self.world > 1
        if self.peer:
            fused_peer_setup(self.slabs[0], dist)
        # owned conducting edges of every rank (rank order), for the all-gather
        owned = self.comm.allgather([s.owned.astype(np.float64) for s in self.slabs])
        self.owned_all = [o.astype(np.int64) for o in owned]
        cover = np.concatenate(self.owned_all) if self.owned_all else np.zeros(0, np.int64)
        if cover.size != self.n_c or not np.array_equal(np.sort(cover), np.arange(self.n_c)):
            raise RuntimeError("owned conducting edges do not partition the conducting block")
        self.a_c = np.zeros(self.n_c)
        self.t = 0.0
        self.pcg_seconds = 0.0
        self._set_state(self.a_c, 0.0)

    def close(self):
        for s in self.slabs:
            s.close()
        self.slabs = []

    # -- state --------------------------------------------------------------
    def _set_state(self, a_c, t):
        self.a_c = np.array(a_c, dtype=np.float64, copy=True)
        self.t = float(t)
        for s in self.slabs:
            s.state_set(self.a_c)

    def set_state(self, a_c, t: float):
        a_c = np.asarray(a_c, np.float64)
        if a_c.shape != (self.n_c,):
            raise ValueError(f"a_c has shape {a_c.shape}, expected ({self.n_c},)")
        self._set_state(a_c, t)

    # -- one solve_kn (schur.py:239-264) --------------------------------------
    def _allreduce(self, parts):
        return self.comm.allreduce(parts)

    def _pcg(self, which: str) -> _lib.SolveReportC:
        """krylov.py:174-250 on the slabs: b = the named rhs, x0 and the
        solution in each slab's x."""
        rep = _lib.SolveReportC()
        t0 = time.perf_counter()
        if self.pcg_mode == "host":
            from .slab import slab_pcg_solve
            for s in self.slabs:
                s.stage_b(which)
            it, relres, conv, app = slab_pcg_solve(self.slabs, self.comm.halo, x0_given=True, rel_tol=self.rel_tol,
                                                   abs_tol=self.abs_tol, max_iter=self.max_iter, jacobi=True)
            rep.iterations, rep.final_rel_residual, rep.converged, rep.applies = it, relres, int(conv), app
            self.pcg_seconds += time.perf_counter() - t0
            return rep
        if self.peer:
            s = self.slabs[0]
            rc = self.lib.mq_slab_fused_solve_peer(s.ctx, ctypes.c_void_p(s.vecs[which]), 1, self.rel_tol,
                                                   self.abs_tol, self.max_iter, 1, ctypes.byref(rep))
        else:
            n = len(self.slabs)
            ctxs = (ctypes.c_void_p * n)(*[s.ctx.value for s in self.slabs])
            bs = (ctypes.c_void_p * n)(*[s.vecs[which] for s in self.slabs])
            xs = (ctypes.c_void_p * n)(*[s.x for s in self.slabs])
            rc = self.lib.mq_slab_fused_solve_local(ctxs, n, bs, xs, 1, self.rel_tol, self.abs_tol,
                                                    self.max_iter, 1, ctypes.byref(rep))
        self.pcg_seconds += time.perf_counter() - t0
        if rc == _lib.MQ_INDEFINITE:
            raise IndefiniteOperatorError(_lib.last_error())
        check(rc, allow=(0, 1))
        return rep

    def solve(self, fam: int, which: int) -> _lib.SolveReportC:
        tots = self._allreduce([s.project(fam, which) for s in self.slabs])
        for s, tot in zip(self.slabs, tots):
            s.start(fam, tot)
        rep = self._pcg("rhs_src" if which == 0 else "rhs_cpl")
        if not rep.converged:
            name = {FAM_SOURCE: "source", FAM_CUR: "coupling_current", FAM_PREV: "coupling_previous"}[fam]
            raise StepFailureError(f"inner solve ({name}) stalled at relative residual "
                                   f"{rep.final_rel_residual:.3e} after {rep.iterations} iterations")
        for s in self.slabs:
            s.store(fam, rep)
        self._observe(fam)
        return rep

    def _observe(self, fam: int):
        if self.strategy == "previous":
            for s in self.slabs:
                s.observe(fam, 0)
            return
        if self.strategy != "cspe":
            return
        tots = self._allreduce([s.observe(fam, 0)[0] for s in self.slabs])
        tots = self._allreduce([s.observe(fam, 1, t)[0] for s, t in zip(self.slabs, tots)])
        tots = self._allreduce([s.observe(fam, 2, t)[0] for s, t in zip(self.slabs, tots)])
        flags = {s.observe(fam, 3, t)[1] for s, t in zip(self.slabs, tots)}
        if len(flags) != 1:
            raise RuntimeError("ranks disagree on a CSPE insert decision")
        if flags.pop():
            self.comm.exchange(self.slabs, ["w2"])
            tots = self._allreduce([s.observe(fam, 4)[0] for s in self.slabs])
            for s, t in zip(self.slabs, tots):
                s.observe(fam, 5, t)

    # -- explicit_euler_step (schur.py:379-405) ------------------------------
    def step(self, dt: float, step_index: int | None = None):
        if dt < 0:
            raise ValueError("dt must be nonnegative")
        wave = self.problem.waveform
        t_new = self.t + dt
        for s in self.slabs:
            s.rhs(0, float(wave(t_new)))
        rep_src = self.solve(FAM_SOURCE, 0)
        for s in self.slabs:
            s.rhs(1)
        rep_cpl = self.solve(FAM_PREV, 1)
        for s in self.slabs:
            s.euler_prep()
        self.comm.exchange(self.slabs, ["dvec"])
        owned_vals = self.comm.allgather([s.euler(dt) for s in self.slabs])
        a_next = np.empty(self.n_c)
        for idx, vals in zip(self.owned_all, owned_vals):
            a_next[idx] = vals
        if not np.isfinite(a_next).all():
            where = f" at step {step_index}" if step_index is not None else ""
            raise StepFailureError(f"non-finite conducting state{where} (t = {t_new:.6e})")
        self._set_state(a_next, t_new)
        return rep_src, rep_cpl

    # -- recover_an (schur.py:408-419) ----------------------------------------
    def recover(self, gather: bool = True):
        wave = self.problem.waveform
        for s in self.slabs:
            s.rhs(0, float(wave(self.t)))
        rep_src = self.solve(FAM_SOURCE, 0)
        for s in self.slabs:
            s.rhs(1)
        rep_cur = self.solve(FAM_CUR, 1)
        return (self.gather_an() if gather else None), (rep_src, rep_cur)

    def gather_an(self) -> np.ndarray:
        """a_n of the last recovery in the reference's compact order (every rank)."""
        parts = self.comm.allgather([np.concatenate([s.gidx.astype(np.float64), s.a_n_local()])
                                     for s in self.slabs])
        a_n = np.zeros(self.n_n)
        for p in parts:
            m = p.size // 2
            a_n[p[:m].astype(np.int64)] = p[m:]
        return a_n

    def diagnostics(self) -> dict:
        d = self.slabs[0].diagnostics()
        return {"basis_cols": list(d.basis_cols), "columns_accepted": list(d.columns_accepted),
                "columns_dropped": list(d.columns_dropped), "evictions": list(d.evictions),
                "maintenance_applies": int(d.maintenance_applies), "pcg_applies": int(d.pcg_applies),
                "solves": list(d.solves), "iterations": list(d.iterations)}


def run_explicit_sharded(problem, n_steps: int, dt: float, *, world: int, dist=None, device: int = 0,
                         strategy: str = "cspe", max_cols: int = 5, rel_tol: float = 1e-8, max_iter: int = 5000,
                         recover_every_step: bool = True, record_states: bool = False,
                         stepper: SlabStepper | None = None) -> ShardedRun:
    """n_steps explicit-Euler steps from a_c = 0 (schur.py:474-607 with a fixed
    dt and an output row per step): per step [src, cpl_prev, src_rec, cpl_cur]
    iterations, optional per-step (a_c, a_n)."""
    own = stepper is None
    st = stepper or SlabStepper(problem, world, dist=dist, device=device, strategy=strategy, max_cols=max_cols,
                                rel_tol=rel_tol, max_iter=max_iter)
    try:
        its = np.zeros((n_steps, 4), dtype=np.int64)
        ac_h = np.zeros((n_steps, st.n_c)) if record_states else None
        an_h = np.zeros((n_steps, st.n_n)) if (record_states and recover_every_step) else None
        a_n = None
        secs = []
        for m in range(n_steps):
            t0 = time.perf_counter()
            r1, r2 = st.step(dt, m + 1)
            its[m, 0], its[m, 1] = r1.iterations, r2.iterations
            if recover_every_step:
                a_n, (r3, r4) = st.recover(gather=record_states or m == n_steps - 1)
                its[m, 2], its[m, 3] = r3.iterations, r4.iterations
            secs.append(time.perf_counter() - t0)
            if record_states:
                ac_h[m] = st.a_c
                if an_h is not None:
                    an_h[m] = a_n
        return ShardedRun(step_iterations=its, final_a_c=st.a_c.copy(), final_a_n=a_n, a_c_history=ac_h,
                          a_n_history=an_h, step_seconds=secs,
                          aggregates={"pcg_seconds": st.pcg_seconds, **st.diagnostics()})
    finally:
        if own:
            st.close()
