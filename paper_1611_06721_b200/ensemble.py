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
