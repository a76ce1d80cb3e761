"""Multi-query ensemble (BASELINE configs[3]) sharded over ranks.

Every member is an independent 64^3 run (config 1 geometry) whose coil
current amplitude J and iron conductivity kappa are scaled by factors drawn
U(0.8, 1.2) from a seed (J factors first, then kappa factors; SURVEY 8(d)
item 9).  K_n is the same for every member (nu is unchanged).  Members are
split into contiguous, balanced blocks over the ranks of one node; there is
no collective on the data path — only the final gather of per-member results
and a max-over-ranks of the timing.  ``torch.distributed`` carries those two
(nccl on GPUs, gloo in the CPU tests).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import configs as C


def shard(n_members: int, world: int, rank: int) -> range:
    """Contiguous balanced block of member indices owned by ``rank``."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("invalid world/rank")
    base, extra = divmod(n_members, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


@dataclass
class MemberResult:
    member: int
    j_factor: float
    kappa_factor: float
    steps: int
    dt: float
    iterations: dict = field(default_factory=dict)
    final_norm_a_c: float = 0.0
    device_ms: float = 0.0


def member_problem(member: int, n_members: int = 256, seed: int = 0):
    j, k = C.ensemble_factors(n_members, seed)
    prob = C.make_problem(3, j_scale=float(j[member]), kappa_scale=float(k[member]))
    # dt_i = dt_nominal * kappa_i / kappa_0 (lambda ~ 1/kappa through M_c)
    dt = C.config_spec(3).dt * float(k[member])
    return prob, float(j[member]), float(k[member]), dt


def run_member(member: int, steps: int, *, n_members: int = 256, seed: int = 0, device: int = 0,
               strategy: str = "cspe", max_cols: int = 5) -> MemberResult:
    """Integrate one member on the local GPU with the device-resident loop."""
    from .krylov import PcgConfig
    from .schur import run_explicit
    prob, jf, kf, dt = member_problem(member, n_members, seed)
    res = run_explicit(prob, t_end=steps * dt, dt=dt, strategy=strategy,
                       pcg=PcgConfig(rel_tol=1e-8, max_iter=5000),
                       output_period=dt * (1 - 1e-3), max_cols=max_cols, device=device)
    return MemberResult(member, jf, kf, res.aggregates["steps"], dt,
                        dict(res.aggregates["iterations"]),
                        float(np.linalg.norm(res.final_a_c)),
                        1000.0 * res.aggregates["wall_seconds"])


def run_members(members, steps: int, *, concurrency: int = 1, n_members: int = 256, seed: int = 0,
                device: int = 0, strategy: str = "cspe", max_cols: int = 5) -> list:
    """Integrate several members on one GPU, ``concurrency`` at a time.

    Each member of a wave has its own context and stream and its PCG kernel
    confined to an equal slice of the SMs (``mq_ctx_set_sm_budget``); the
    waves' step graphs are enqueued interleaved, so the members' kernels run
    side by side (the single-member PCG at 64^3 is latency-bound and leaves
    the chip under-used).  Same trajectory per member as :func:`run_member`
    up to the reduction order of the dot products (grid size).

    Measured on B200 at 64^3 (10 steps): one member on the whole GPU with the
    shared-memory-resident PCG kernel 279 steps/s; 4 members side by side on
    37-SM slices (TMA brick kernel) 248 member-steps/s.  Hence the default
    concurrency 1; slices pay off only for grids too large for the resident
    kernel and too small to fill the chip."""
    import ctypes
    import time

    from . import _lib
    from ._lib import check, dptr
    from .krylov import PcgConfig
    from .schur import SchurOperator, StepFailureError, recover_an
    from .startvec import RhsFamily
    members = list(members)
    sms = _lib.sm_count(device)
    out = []
    for w0 in range(0, len(members), max(1, concurrency)):
        wave = members[w0:w0 + max(1, concurrency)]
        runs = []
        for m in wave:
            prob, jf, kf, dt = member_problem(m, n_members, seed)
            op = SchurOperator(prob, pcg=PcgConfig(rel_tol=1e-8, max_iter=5000), strategy=strategy,
                               max_cols=max_cols, device=device)
            if len(wave) > 1:
                op.grid.set_sm_budget(sms // len(wave))
            a0 = np.zeros(op.grid.n_c)
            _, (r1, r2) = recover_an(op, a0, 0.0)
            op._set_state(a0, 0.0)
            tt = [0.0]
            for _ in range(steps):
                tt.append(tt[-1] + dt)
            wave_tab = np.array([float(prob.waveform(t)) for t in tt])
            check(op.lib.mq_run_prepare(op.grid.ctx, steps, dptr(np.full(steps, dt)), dptr(wave_tab), 1))
            runs.append((m, jf, kf, dt, op, r1.iterations, r2.iterations))
        t0 = time.perf_counter()
        for _ in range(steps):
            for (_, _, _, _, op, _, _) in runs:
                check(op.lib.mq_run_steps(op.grid.ctx, 1, 1, None))
        for (_, _, _, _, op, _, _) in runs:
            op.grid.sync()
        wall_ms = 1000.0 * (time.perf_counter() - t0)
        for (m, jf, kf, dt, op, i_src0, i_cur0) in runs:
            it = np.zeros((steps, 4), dtype=np.int32)
            failed = ctypes.c_int64(-1)
            rc = op.lib.mq_run_finish(op.grid.ctx, _lib.i32ptr(it), ctypes.byref(failed))
            if rc == _lib.MQ_NONFINITE:
                raise StepFailureError(f"member {m}: non-finite conducting state at step {failed.value}")
            check(rc)
            iters = {RhsFamily.SOURCE_CURRENT.value: int(i_src0 + it[:, 0].sum() + it[:, 2].sum()),
                     RhsFamily.COUPLING_FROM_PREVIOUS_STATE.value: int(it[:, 1].sum()),
                     RhsFamily.COUPLING_FROM_CURRENT_STATE.value: int(i_cur0 + it[:, 3].sum())}
            a_c = op._get_state()
            out.append(MemberResult(m, jf, kf, steps, dt, iters, float(np.linalg.norm(a_c)),
                                    wall_ms / len(runs)))
            op.grid.close()
    return out


def gather_results(local: list, dist=None) -> list:
    """All-gather per-member results (object lists) over the ranks."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return sorted(local, key=lambda r: r.member)
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, local)
    return sorted((r for part in out for r in part), key=lambda r: r.member)


def max_over_ranks(value: float, dist=None, device=None) -> float:
    """Max of a per-rank timing (the job's wall time is the slowest rank)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64,
                     device=device if device is not None else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
