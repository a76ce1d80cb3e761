"""Device twins of the reference's Schur/explicit-Euler entry points.

``SchurOperator.solve_kn`` (schur.py:239-264), ``explicit_euler_step``
(schur.py:379-405), ``recover_an`` (schur.py:408-419) and ``run_explicit``
(schur.py:474-607) keep the reference's names, arguments, counters and
exceptions; underneath, the conducting state, the three right-hand-side
families, their start-vector histories and every PCG solve stay on the GPU.
``run_explicit`` runs the whole time loop on the device (one CUDA graph per
step, replayed) and synchronises with the host only at output rows that need
host data, or once at the end.

The reference's other ``SchurOperator`` options are honoured as it defines
them: ``strategy=<StartVectorStrategy object>`` (any object with the
protocol of startvec.py:315-342, e.g. the reference's own ``CspeStrategy``;
schur.py:198-199), ``cache_source_solve`` (one pattern solve rescaled per
call, schur.py:266-278) and ``projection_target`` (schur.py:244-250).  With
a host-side strategy object or a cached source solve the step is composed on
the host from device operations (PCG, K_cn, K_cn^T, K_c products), exactly
the reference's sequence (schur.py:379-419, 474-607); otherwise the whole
step runs on the device.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import check, dptr, f64, i64ptr
from .device import DeviceGrid, Problem, default_probe_cells
from .krylov import JacobiPreconditioner, PcgConfig, Preconditioner, SolveReport, pcg_solve
from .startvec import DeviceStrategy, RhsFamily, family_index, solver_cfg

__all__ = ["StepFailureError", "SchurOperator", "explicit_euler_step", "recover_an",
           "run_explicit", "TransientResult", "FAMILIES", "step_times", "CflEstimate", "trace_bytes",
           "estimate_cfl"]

FAMILIES = (RhsFamily.SOURCE_CURRENT, RhsFamily.COUPLING_FROM_CURRENT_STATE,
            RhsFamily.COUPLING_FROM_PREVIOUS_STATE)


class StepFailureError(RuntimeError):
    """Non-finite state or a stalled inner solve (schur.py:56-57)."""


def _report(r: _lib.SolveReportC) -> SolveReport:
    return SolveReport(int(r.iterations), float(r.final_rel_residual), bool(r.converged),
                       int(r.applies))


class _DeviceStrategyView:
    """``op.strategy`` of an operator whose strategy runs on the device:
    the reference's strategy queries (startvec.py:315-342) answered from the
    device diagnostics."""

    def __init__(self, op):
        self._op = op
        self.kind = op.strategy_kind

    def basis_size(self, family=None) -> int:
        if family is not None and self.kind == "cspe":
            return int(self._op.diagnostics().basis_cols[family_index(family)])
        return self._op.basis_size()

    @property
    def maintenance_applies(self) -> int:
        return self._op.maintenance_applies

    def diagnostics(self) -> dict:
        return self._op.strategy_diagnostics()


class SchurOperator:
    """Device-resident eliminated-block operator (schur.py:168-313)."""

    def __init__(self, problem, pcg: PcgConfig | None = None, strategy="previous", *,
                 preconditioner=Preconditioner.JACOBI, cache_source_solve: bool = False,
                 projection_target: str = "assembled-rhs", max_cols: int = 20,
                 n_pod: int = 10, eps_pod: float = 1e-4, device: int = 0):
        if projection_target not in ("assembled-rhs", "composed-coupling"):
            raise ValueError(f"unknown projection target {projection_target!r}")
        if Preconditioner(preconditioner) is not Preconditioner.JACOBI:
            raise NotImplementedError("the device K_n path uses the reference's Jacobi preconditioner")
        self.grid = problem if isinstance(problem, DeviceGrid) else DeviceGrid(problem, device)
        self.problem = self.grid.problem
        self.pcg = pcg or PcgConfig()
        self.projection_target = projection_target
        self.cache_source_solve = bool(cache_source_solve)
        self._cached_pattern_solution = None
        # strategy: a name (device solver), a DeviceStrategy on this grid (its
        # device solver and parameters), or any StartVectorStrategy-protocol
        # object, which stays on the host (schur.py:198-199)
        self.host_strategy = None
        if isinstance(strategy, DeviceStrategy) and strategy.grid is self.grid:
            max_cols, n_pod, eps_pod = strategy.max_cols, strategy.n_pod, strategy.eps_pod
            self.strategy_kind = strategy.kind
        elif isinstance(strategy, str):
            self.strategy_kind = strategy.lower()
        else:
            if not (hasattr(strategy, "start_vector") and hasattr(strategy, "observe")):
                raise ValueError(f"strategy must be a name or a StartVectorStrategy, got {strategy!r}")
            self.host_strategy = strategy
            self.strategy_kind = str(getattr(strategy, "kind", "custom"))
        # composed: the step is built on the host from device operations
        self.composed = self.host_strategy is not None or self.cache_source_solve
        if self.problem.pattern is None:
            raise ValueError("problem has no source pattern")
        pat = f64(self.problem.pattern, self.grid.n_n, "source pattern")
        cfg = solver_cfg("zero" if self.host_strategy is not None else self.strategy_kind, max_cols=max_cols,
                         n_pod=n_pod, eps_pod=eps_pod, rel_tol=self.pcg.rel_tol, abs_tol=self.pcg.abs_tol,
                         max_iter=self.pcg.max_iter, drop_tol=self.pcg.rel_tol)
        self.cfg = cfg
        self.lib = self.grid.lib
        check(self.lib.mq_solver_init(self.grid.ctx, ctypes.byref(cfg), dptr(pat)))
        self.solve_iterations = {f: [] for f in FAMILIES}
        self.solver_seconds = 0.0
        self._host_applies = 0
        self._rhs = self.grid.alloc()
        self._y = self.grid.alloc()
        self._kn = self.grid.kn_operator()
        self._jac = JacobiPreconditioner(self._kn.diagonal())   # schur.py:193-197
        self._minv_diag = 1.0 / self.grid.mc_diag()
        self.t = 0.0
        # page-locked result arrays of the host-facing step / recovery calls,
        # allocated now rather than inside the first steps
        _lib.pinned_reserve(self.grid.n_c, 4)
        _lib.pinned_reserve(self.grid.n_n, 4)

    @property
    def strategy(self):
        """The host strategy object, or a DeviceStrategy-like view of the
        device solver (basis_size / diagnostics)."""
        return self.host_strategy if self.host_strategy is not None else _DeviceStrategyView(self)

    @property
    def system_n_c(self):
        return self.grid.n_c

    def diagnostics(self) -> _lib.Diag:
        d = _lib.Diag()
        check(self.lib.mq_diagnostics(self.grid.ctx, ctypes.byref(d)))
        return d

    @property
    def pcg_applies(self) -> int:
        return int(self.diagnostics().pcg_applies) + self._host_applies

    @property
    def maintenance_applies(self) -> int:
        if self.host_strategy is not None:
            return int(getattr(self.host_strategy, "maintenance_applies", 0))
        return int(self.diagnostics().maintenance_applies)

    def solve_count(self, family) -> int:
        return len(self.solve_iterations[family])

    def total_solves(self) -> int:
        return sum(len(v) for v in self.solve_iterations.values())

    def total_iterations(self) -> int:
        return sum(sum(v) for v in self.solve_iterations.values())

    def basis_size(self) -> int:
        if self.host_strategy is not None:
            return int(self.host_strategy.basis_size())
        d = self.diagnostics()
        if self.strategy_kind == "cspe":
            return int(max(d.basis_cols))
        if self.strategy_kind == "pod":
            return int(d.pod_k)
        return 0

    def strategy_diagnostics(self) -> dict:
        if self.host_strategy is not None:
            diag = getattr(self.host_strategy, "diagnostics", None)
            return dict(diag()) if diag else {}
        d = self.diagnostics()
        if self.strategy_kind == "cspe":
            return {"basis_cols": int(max(d.basis_cols)),
                    "maintenance_applies": int(d.maintenance_applies)}
        if self.strategy_kind == "pod":
            return {"pod_k": int(d.pod_k), "pod_info": float(d.pod_info),
                    "min_pod_info": float(d.min_pod_info),
                    "maintenance_applies": int(d.maintenance_applies)}
        return {}

    def solve_kn(self, rhs, family, raw_state=None) -> tuple[np.ndarray, SolveReport]:
        """One pseudo-inverse action K_n^+ rhs for the family (schur.py:239-264)."""
        started = time.perf_counter()
        fam = family if isinstance(family, RhsFamily) else RhsFamily(getattr(family, "value", family))
        if self.host_strategy is not None:
            target = rhs
            if (self.projection_target == "composed-coupling" and raw_state is not None
                    and fam is not RhsFamily.SOURCE_CURRENT):
                # schur.py:244-250: the target recomposed from the coupling operator
                target = self.grid.kcn_t_apply(raw_state)
            x0 = self.host_strategy.start_vector(family, target)
            y, rep = pcg_solve(self._kn, rhs, x0=x0, config=self.pcg, preconditioner=self._jac)
            if not rep.converged:
                raise StepFailureError(f"inner solve ({fam.value}) stalled at relative residual "
                                       f"{rep.final_rel_residual:.3e} after {rep.iterations} iterations")
            self._host_applies += rep.applications
            self.host_strategy.observe(family, y)
        else:
            # the device solver projects onto the assembled rhs; the composed
            # coupling target is the same vector (K_cn^T a_c, schur.py:246-249)
            self.grid.upload(f64(rhs, self.grid.n_n, "rhs"), self._rhs)
            r = _lib.SolveReportC()
            rc = self.lib.mq_solve_kn(self.grid.ctx, family_index(family), ctypes.c_void_p(self._rhs),
                                      ctypes.c_void_p(self._y), ctypes.byref(r))
            check(rc)
            y = self.grid.download(self._y)
            rep = _report(r)
        self.solve_iterations[fam].append(int(rep.iterations))
        self.solver_seconds += time.perf_counter() - started
        return y, rep

    def source_solution(self, t: float):
        """K_n^+ j_n(t); with cache_source_solve one pattern solve, rescaled
        per call (schur.py:266-278)."""
        scale = float(self.problem.waveform(t))
        if self.cache_source_solve:
            if self._cached_pattern_solution is None:
                y, rep = self.solve_kn(self.problem.pattern, RhsFamily.SOURCE_CURRENT)
                self._cached_pattern_solution = y
            else:
                rep = SolveReport(0, 0.0, True)
            return self._cached_pattern_solution * scale, rep
        return self.solve_kn(self.problem.pattern * scale, RhsFamily.SOURCE_CURRENT)

    def apply(self, x, lin_state, family=RhsFamily.COUPLING_FROM_PREVIOUS_STATE) -> np.ndarray:
        """K_S(lin_state) x, charging the inner solve to ``family`` (schur.py:289-296)."""
        w = self.grid.kcn_t_apply(x)
        y, _ = self.solve_kn(w, family, raw_state=x)
        return self.grid.kc_apply(lin_state, x) - self.grid.kcn_apply(y)

    def apply_detached(self, x, lin_state, inner_start=None):
        """K_S x with an explicit inner start vector and no family history
        (schur.py:298-313); returns (K_S x, inner solution)."""
        started = time.perf_counter()
        w = self.grid.kcn_t_apply(x)
        y, rep = pcg_solve(self._kn, w, x0=inner_start, config=self.pcg, preconditioner=self._jac)
        if not rep.converged:
            raise StepFailureError("spectral probe solve stalled")
        self._host_applies += rep.applications
        self.solver_seconds += time.perf_counter() - started
        return self.grid.kc_apply(lin_state, x) - self.grid.kcn_apply(y), y

    def minv(self, x):
        return self._minv_diag * x

    def _set_state(self, a_c, t):
        v = f64(a_c, self.grid.n_c, "state")
        check(self.lib.mq_state_set(self.grid.ctx, dptr(v), float(t)))
        self.t = float(t)

    def _get_state(self):
        out = np.empty(self.grid.n_c)
        check(self.lib.mq_state_get(self.grid.ctx, dptr(out), None))
        return out

    def set_probe(self, cells=None) -> np.ndarray:
        """Device B probe over ``cells`` (global conductor-cell ids; default
        model.py:562-566).  Every later device step logs B_probe."""
        cells = default_probe_cells(self.problem.material) if cells is None else \
            np.ascontiguousarray(cells, dtype=np.int64)
        if cells.size == 0:
            raise ValueError("probe cell set is empty")
        check(self.lib.mq_probe_set(self.grid.ctx, i64ptr(cells), int(cells.size)))
        self.probe_cells = cells
        return cells

    def probe_b(self, a_c=None) -> float:
        """Mean |B| over the probe cells of ``a_c`` (default: the device
        state), model.py:415-425."""
        out = ctypes.c_double()
        arg = dptr(f64(a_c, self.grid.n_c, "state")) if a_c is not None else None
        check(self.lib.mq_probe_b(self.grid.ctx, arg, ctypes.byref(out)))
        return float(out.value)


@dataclass(frozen=True)
class CflEstimate:
    """Largest stable explicit step dt_max = safety * 2 / lambda_max (schur.py:316-324)."""

    lambda_max: float
    dt_max: float
    safety: float
    power_iters: int
    power_tol: float
    pcg_applies: int = 0


def estimate_cfl(op: SchurOperator, a_c_ref=None, *, power_iters: int = 200,
                 power_tol: float = 1e-4, safety: float = 0.9, seed: int = 42,
                 v0=None) -> CflEstimate:
    """lambda_max(M_c^-1 K_S) by power iteration on the device (schur.py:327-376).

    Same start vector rule as the reference (a valid v0, else
    ``default_rng(seed).standard_normal``, normalised); the inner K_n solves are
    device PCG solves warm-started from the previous inner solution.
    """
    if not (0.0 < safety <= 1.0):
        raise ValueError("safety must lie in (0, 1]")
    if power_iters < 1:
        raise ValueError("power_iters must be at least 1")
    n = op.grid.n_c
    ref = None if a_c_ref is None else f64(a_c_ref, n, "reference state")
    v = None
    if v0 is not None:
        v = np.asarray(v0, dtype=np.float64).copy()
        if v.shape != (n,) or not np.linalg.norm(v) > 0.0:
            v = None
        else:
            v = v / np.linalg.norm(v)
    if v is None:
        v = np.random.default_rng(seed).standard_normal(n)
        v /= np.linalg.norm(v)
    v = np.ascontiguousarray(v)
    lam, dt = ctypes.c_double(), ctypes.c_double()
    used, applies = ctypes.c_int32(), ctypes.c_int64()
    rc = op.lib.mq_estimate_cfl(op.grid.ctx, dptr(ref) if ref is not None else None, dptr(v),
                                int(power_iters), float(power_tol), float(safety),
                                float(op.pcg.rel_tol), int(op.pcg.max_iter), ctypes.byref(lam),
                                ctypes.byref(dt), ctypes.byref(used), ctypes.byref(applies))
    check(rc)
    return CflEstimate(lam.value, dt.value, safety, int(used.value), power_tol, int(applies.value))


def _composed_euler_step(state, dt, op, step_index):
    """schur.py:379-405 composed on the host from device operations (a host
    strategy object or a cached source solve)."""
    a_c, t = state
    a_c = f64(a_c, op.grid.n_c, "state")
    t_new = t + dt
    y_src, rep_src = op.source_solution(t_new)
    w = op.grid.kcn_t_apply(a_c)
    y_cpl, rep_cpl = op.solve_kn(w, RhsFamily.COUPLING_FROM_PREVIOUS_STATE, raw_state=a_c)
    rate = op.grid.kcn_apply(y_cpl - y_src) - op.grid.kc_apply(a_c, a_c)
    a_next = a_c + dt * op.minv(rate)
    if not np.isfinite(a_next).all():
        where = f" at step {step_index}" if step_index is not None else ""
        raise StepFailureError(f"non-finite conducting state{where} (t = {t_new:.6e})")
    op.t = float(t_new)
    return a_next, (rep_src, rep_cpl)


def _composed_recover_an(op, a_c, t):
    """schur.py:408-419 composed on the host from device operations."""
    a_c = f64(a_c, op.grid.n_c, "state")
    y_src, rep_src = op.source_solution(t)
    w = op.grid.kcn_t_apply(a_c)
    y_cpl, rep_cpl = op.solve_kn(w, RhsFamily.COUPLING_FROM_CURRENT_STATE, raw_state=a_c)
    op.t = float(t)
    return y_src - y_cpl, (rep_src, rep_cpl)


def explicit_euler_step(state, dt: float, op: SchurOperator, step_index: int | None = None):
    """One explicit Euler step on the device (schur.py:379-405)."""
    a_c, t = state
    if dt < 0:
        raise ValueError("dt must be nonnegative")
    if op.composed:
        return _composed_euler_step(state, dt, op, step_index)
    started = time.perf_counter()
    v = f64(a_c, op.grid.n_c, "state")
    t_new = t + dt
    a_next = _lib.pinned_empty(op.grid.n_c)
    r1, r2 = _lib.SolveReportC(), _lib.SolveReportC()
    rc = op.lib.mq_euler_step_host(op.grid.ctx, dptr(v), float(t), float(dt), float(op.problem.waveform(t_new)),
                                   int(step_index if step_index is not None else -1), dptr(a_next),
                                   ctypes.byref(r1), ctypes.byref(r2))
    op.t = float(t)
    if rc == _lib.MQ_NONFINITE:
        where = f" at step {step_index}" if step_index is not None else ""
        raise StepFailureError(f"non-finite conducting state{where} (t = {t_new:.6e})")
    check(rc)
    op.solve_iterations[RhsFamily.SOURCE_CURRENT].append(int(r1.iterations))
    op.solve_iterations[RhsFamily.COUPLING_FROM_PREVIOUS_STATE].append(int(r2.iterations))
    op.t = float(t_new)
    op.solver_seconds += time.perf_counter() - started
    return a_next, (_report(r1), _report(r2))


def recover_an(op: SchurOperator, a_c, t: float):
    """a_n = K_n^+ j_n(t) - K_n^+ K_cn^T a_c (schur.py:408-419)."""
    if op.composed:
        return _composed_recover_an(op, a_c, t)
    started = time.perf_counter()
    v = f64(a_c, op.grid.n_c, "state")
    a_n = _lib.pinned_empty(op.grid.n_n)
    r1, r2 = _lib.SolveReportC(), _lib.SolveReportC()
    rc = op.lib.mq_recover_an_host(op.grid.ctx, dptr(v), float(t), float(op.problem.waveform(t)), dptr(a_n),
                                   ctypes.byref(r1), ctypes.byref(r2))
    op.t = float(t)
    check(rc)
    op.solve_iterations[RhsFamily.SOURCE_CURRENT].append(int(r1.iterations))
    op.solve_iterations[RhsFamily.COUPLING_FROM_CURRENT_STATE].append(int(r2.iterations))
    op.solver_seconds += time.perf_counter() - started
    return a_n, (_report(r1), _report(r2))


@dataclass
class TransientResult:
    """schur.py:422-443."""

    times: np.ndarray
    probe_b: np.ndarray
    iters_src: np.ndarray
    iters_cpl_prev: np.ndarray
    iters_cpl_cur: np.ndarray
    basis_cols: np.ndarray
    pod_k: np.ndarray
    pod_info: np.ndarray
    final_a_c: np.ndarray
    final_a_n: np.ndarray | None
    aggregates: dict = field(default_factory=dict)
    step_iterations: np.ndarray | None = None   # per step [src, prev, src_rec, cur]
    a_c_history: np.ndarray | None = None       # record_states: a_c after every step
    a_n_history: np.ndarray | None = None       # record_states: a_n recovered after every step

    @property
    def n_rows(self) -> int:
        return self.times.size


def step_times(t_end: float, dt: float, output_period: float, max_steps: int = 2_000_000):
    """The reference loop's (step_dt list, output-after-step flags)
    (schur.py:546-572) for a fixed dt."""
    dts, outs, _ = _Schedule(t_end, output_period, max_steps).take(dt)
    return dts, outs


class _Schedule:
    """The reference loop's step sizes and output flags (schur.py:546-572),
    produced on the host in the same float order, a phase at a time (the
    step size may shrink between phases when dt="auto" re-estimates)."""

    def __init__(self, t_end: float, output_period: float, max_steps: int):
        self.t_end, self.period, self.max_steps = t_end, output_period, max_steps
        self.eps = 1e-12 * t_end
        self.t = 0.0
        self.next_output = output_period
        self.count = 0

    @property
    def done(self) -> bool:
        return not (self.t < self.t_end - self.eps)

    def take(self, dt: float, nmax=None):
        """(step sizes, output flags, node times incl. the start) of up to
        nmax further steps of size dt."""
        dts, outs, tt = [], [], [self.t]
        while not self.done and (nmax is None or len(dts) < nmax):
            step_dt = min(dt, self.t_end - self.t)
            self.t += step_dt
            self.count += 1
            if self.count > self.max_steps:
                raise StepFailureError(f"step budget exceeded ({self.max_steps})")
            out = self.t >= self.next_output - self.eps or self.t >= self.t_end - self.eps
            if out:
                while self.next_output <= self.t + self.eps:
                    self.next_output += self.period
            dts.append(step_dt)
            outs.append(out)
            tt.append(self.t)
        return dts, outs, tt


def run_explicit(problem, t_end: float, dt, *, strategy="cspe", pcg: PcgConfig | None = None,
                 preconditioner=Preconditioner.JACOBI, output_period: float = 1e-3,
                 probe=None, a0=None, max_cols: int = 20, n_pod: int = 10,
                 eps_pod: float = 1e-4, max_steps: int = 2_000_000, device: int = 0,
                 use_graph: bool = True, record_states: bool = False,
                 op: SchurOperator | None = None, reestimate_every: int = 500, safety: float = 0.9,
                 power_iters: int = 200, power_tol: float = 1e-4,
                 seed: int = 42, cache_source_solve: bool = False,
                 projection_target: str = "assembled-rhs") -> TransientResult:
    """Integrate with explicit Euler on the device (schur.py:474-607).

    ``dt="auto"`` runs the device spectral estimate before the loop and again
    every ``reestimate_every`` steps at the current state, shrinking the step
    when the bound tightened (a fixed dt is never adjusted), as the reference.
    The steps between outputs run as one device-resident sequence (one CUDA
    graph per step).
    """
    if t_end <= 0:
        raise ValueError("t_end must be positive")
    if output_period <= 0:
        raise ValueError("output_period must be positive")
    wall_start = time.perf_counter()
    if op is None:
        op = SchurOperator(problem, pcg=pcg, strategy=strategy, preconditioner=preconditioner,
                           cache_source_solve=cache_source_solve, projection_target=projection_target,
                           max_cols=max_cols, n_pod=n_pod, eps_pod=eps_pod, device=device)
    if op.composed:
        return _run_composed(op, t_end, dt, output_period=output_period, probe=probe, a0=a0,
                             max_steps=max_steps, reestimate_every=reestimate_every, safety=safety,
                             power_iters=power_iters, power_tol=power_tol, seed=seed, wall_start=wall_start)
    lambda_max = None
    auto = isinstance(dt, str)
    if auto:
        if dt != "auto":
            raise ValueError(f"dt must be a number or 'auto', got {dt!r}")
        est = estimate_cfl(op, power_iters=power_iters, power_tol=power_tol, safety=safety, seed=seed)
        dt, lambda_max = est.dt_max, est.lambda_max
    dt = float(dt)
    if dt <= 0:
        raise ValueError("dt must be positive")
    n_c = op.grid.n_c
    # probe: a host callable (a_c, a_n, t) -> float as in the reference, or
    # "device" / an array of conductor-cell ids for the device probe, which
    # logs B_probe inside the step graph
    host_probe = callable(probe)
    device_probe = probe is not None and not host_probe
    if device_probe:
        if isinstance(probe, str):
            if probe != "device":
                raise ValueError(f"probe must be a callable, 'device' or cell ids, got {probe!r}")
            op.set_probe()
        else:
            op.set_probe(probe)
    a_c = np.zeros(n_c) if a0 is None else f64(a0, n_c, "initial state").copy()
    wave = op.problem.waveform
    rows = {k: [] for k in ("t", "b", "src", "prev", "cur", "basis", "k", "info")}

    def emit(t_row, a_c_row, a_n_row, iters_src, iters_prev, iters_cur, pod_window=()):
        # pod_window: the (pod_k, pod_info) samples the reference's
        # _WindowStats.note_pod took after each Euler step since the last row
        rows["t"].append(t_row)
        if host_probe:
            rows["b"].append(float(probe(a_c_row, a_n_row, t_row)))
        else:
            rows["b"].append(op.probe_b(a_c_row) if device_probe else 0.0)
        rows["src"].append(float(np.mean(iters_src)) if len(iters_src) else 0.0)
        rows["prev"].append(float(np.mean(iters_prev)) if len(iters_prev) else 0.0)
        rows["cur"].append(float(np.mean(iters_cur)) if len(iters_cur) else 0.0)
        diag = op.strategy_diagnostics()
        rows["basis"].append(op.basis_size())
        if op.strategy_kind == "pod":
            samples = list(pod_window) + [(diag["pod_k"], diag["pod_info"])]
            rows["k"].append(max(k for k, _ in samples))
            rows["info"].append(min([1.0] + [i for _, i in samples]))
        else:
            rows["k"].append(0)
            rows["info"].append(1.0)

    # initial recovery at t = 0 (schur.py:540-541)
    a_n, (r1, r2) = recover_an(op, a_c, 0.0)
    emit(0.0, a_c, a_n, [r1.iterations], [], [r2.iterations])
    op._set_state(a_c, 0.0)
    sched = _Schedule(t_end, output_period, max_steps)
    phase_len = reestimate_every if (auto and reestimate_every > 0) else None
    iters_parts, hist_parts, hist_n_parts = [], [], []
    all_out_all = True
    refreshes = 0
    while not sched.done:
        if phase_len is not None and sched.count > 0 and sched.count % phase_len == 0:
            # schur.py:548-557: re-estimate at the current state, shrink only
            est = estimate_cfl(op, a_c_ref=a_c, power_iters=power_iters, power_tol=power_tol,
                               safety=safety, seed=seed)
            refreshes += 1
            lambda_max = est.lambda_max
            dt = min(dt, est.dt_max)
            op._set_state(a_c, sched.t)
        base = sched.count
        dts, outs, tt = sched.take(dt, phase_len)
        ph0 = time.perf_counter()
        a_c, a_n_ph, step_iters, hist, all_out = _run_phase(
            op, dts, outs, tt, wave, emit, rows, base, host_probe, device_probe, use_graph, record_states)
        # the device phases are solver work (every step is its inner solves
        # plus the n_c-sized Euler update)
        op.solver_seconds += time.perf_counter() - ph0
        if a_n_ph is not None:
            a_n = a_n_ph
        all_out_all = all_out_all and all_out
        iters_parts.append(step_iters)
        if hist is not None:
            hist_parts.append(hist[0])
            hist_n_parts.append(hist[1])
    n = sched.count
    wall = time.perf_counter() - wall_start
    d = op.diagnostics()
    aggregates = {
        "integrator": "explicit",
        "strategy": op.strategy_kind,
        "steps": n,
        "dt": dt,
        "lambda_max": lambda_max,
        "cfl_refreshes": refreshes,
        "solves": {f.value: op.solve_count(f) for f in FAMILIES},
        "iterations": {f.value: int(sum(op.solve_iterations[f])) for f in FAMILIES},
        "mean_iterations": {f.value: (float(np.mean(op.solve_iterations[f]))
                                      if op.solve_iterations[f] else 0.0) for f in FAMILIES},
        "pcg_applies": int(d.pcg_applies),
        "maintenance_applies": int(d.maintenance_applies),
        "operator_applies": int(d.pcg_applies + d.maintenance_applies),
        "wall_seconds": wall,
        "solver_seconds": op.solver_seconds,
        "min_pod_info": float(d.min_pod_info),
        "max_basis_cols": int(max(d.basis_cols)),
        "aborted": False,
    }
    step_iters = (np.concatenate(iters_parts) if iters_parts else np.zeros((0, 4), dtype=np.int32))
    return TransientResult(times=np.asarray(rows["t"]), probe_b=np.asarray(rows["b"]),
                           iters_src=np.asarray(rows["src"]), iters_cpl_prev=np.asarray(rows["prev"]),
                           iters_cpl_cur=np.asarray(rows["cur"]),
                           basis_cols=np.asarray(rows["basis"], dtype=np.int64),
                           pod_k=np.asarray(rows["k"], dtype=np.int64),
                           pod_info=np.asarray(rows["info"]), final_a_c=a_c, final_a_n=a_n,
                           aggregates=aggregates,
                           step_iterations=step_iters if all_out_all and not host_probe else None,
                           a_c_history=np.concatenate(hist_parts) if record_states and hist_parts else
                           (np.empty((0, n_c)) if record_states else None),
                           a_n_history=np.concatenate(hist_n_parts) if record_states and hist_n_parts else
                           (np.empty((0, op.grid.n_n)) if record_states else None))


def _run_composed(op, t_end, dt, *, output_period, probe, a0, max_steps, reestimate_every, safety,
                  power_iters, power_tol, seed, wall_start):
    """The reference's loop (schur.py:474-607, _WindowStats 448-467) over the
    composed step, for operators with a host strategy object or a cached
    source solve."""
    auto = isinstance(dt, str)
    lambda_max = None
    if auto:
        if dt != "auto":
            raise ValueError(f"dt must be a number or 'auto', got {dt!r}")
        est = estimate_cfl(op, power_iters=power_iters, power_tol=power_tol, safety=safety, seed=seed)
        dt_val, lambda_max = est.dt_max, est.lambda_max
    else:
        dt_val = float(dt)
        if dt_val <= 0:
            raise ValueError("dt must be positive")
    n_c = op.grid.n_c
    a_c = np.zeros(n_c) if a0 is None else f64(a0, n_c, "initial state").copy()
    t = 0.0
    if probe is not None and not callable(probe):
        # "device" or conductor-cell ids: the device B probe of each row's state
        op.set_probe(None if isinstance(probe, str) else probe)
        probe = (lambda a, _n, _t: op.probe_b(a))
    rows = {k: [] for k in ("t", "b", "src", "prev", "cur", "basis", "k", "info")}
    win = {f: [] for f in FAMILIES}
    pod = {"k": 0, "info": 1.0}

    def note_pod():
        diag = op.strategy_diagnostics()
        if "pod_k" in diag:
            pod["k"] = max(pod["k"], diag["pod_k"])
            pod["info"] = min(pod["info"], diag.get("pod_info", 1.0))

    def mean(f):
        return float(np.mean(win[f])) if win[f] else 0.0

    def emit_row(t_row, a_n, reps):
        if reps is not None:
            win[RhsFamily.SOURCE_CURRENT].append(reps[0].iterations)
            win[RhsFamily.COUPLING_FROM_CURRENT_STATE].append(reps[1].iterations)
        note_pod()
        rows["t"].append(t_row)
        rows["b"].append(float(probe(a_c, a_n, t_row)) if probe else 0.0)
        rows["src"].append(mean(RhsFamily.SOURCE_CURRENT))
        rows["prev"].append(mean(RhsFamily.COUPLING_FROM_PREVIOUS_STATE))
        rows["cur"].append(mean(RhsFamily.COUPLING_FROM_CURRENT_STATE))
        rows["basis"].append(op.basis_size())
        rows["k"].append(max(pod["k"], op.strategy_diagnostics().get("pod_k", 0)))
        rows["info"].append(pod["info"])
        for f in FAMILIES:
            win[f] = []
        pod["k"], pod["info"] = 0, 1.0

    a_n, reps = recover_an(op, a_c, t)
    emit_row(t, a_n, reps)
    next_output = output_period
    steps = refreshes = 0
    eps = 1e-12 * t_end
    while t < t_end - eps:
        if auto and reestimate_every > 0 and steps > 0 and steps % reestimate_every == 0:
            est = estimate_cfl(op, a_c_ref=a_c, power_iters=power_iters, power_tol=power_tol,
                               safety=safety, seed=seed)
            refreshes += 1
            lambda_max = est.lambda_max
            dt_val = min(dt_val, est.dt_max)
        step_dt = min(dt_val, t_end - t)
        a_c, sreps = explicit_euler_step((a_c, t), step_dt, op, step_index=steps + 1)
        win[RhsFamily.SOURCE_CURRENT].append(sreps[0].iterations)
        win[RhsFamily.COUPLING_FROM_PREVIOUS_STATE].append(sreps[1].iterations)
        note_pod()
        t += step_dt
        steps += 1
        if steps > max_steps:
            raise StepFailureError(f"step budget exceeded ({max_steps})")
        if t >= next_output - eps or t >= t_end - eps:
            a_n, reps = recover_an(op, a_c, t)
            emit_row(t, a_n, reps)
            while next_output <= t + eps:
                next_output += output_period
    diag = op.strategy_diagnostics()
    aggregates = {
        "integrator": "explicit",
        "strategy": op.strategy_kind,
        "steps": steps,
        "dt": dt_val,
        "lambda_max": lambda_max,
        "cfl_refreshes": refreshes,
        "solves": {f.value: op.solve_count(f) for f in FAMILIES},
        "iterations": {f.value: int(sum(op.solve_iterations[f])) for f in FAMILIES},
        "mean_iterations": {f.value: (float(np.mean(op.solve_iterations[f]))
                                      if op.solve_iterations[f] else 0.0) for f in FAMILIES},
        "pcg_applies": op.pcg_applies,
        "maintenance_applies": op.maintenance_applies,
        "operator_applies": op.pcg_applies + op.maintenance_applies,
        "wall_seconds": time.perf_counter() - wall_start,
        "solver_seconds": op.solver_seconds,
        "min_pod_info": diag.get("min_pod_info", 1.0),
        "max_basis_cols": diag.get("basis_cols", 0),
        "aborted": False,
    }
    return TransientResult(times=np.asarray(rows["t"]), probe_b=np.asarray(rows["b"]),
                           iters_src=np.asarray(rows["src"]), iters_cpl_prev=np.asarray(rows["prev"]),
                           iters_cpl_cur=np.asarray(rows["cur"]),
                           basis_cols=np.asarray(rows["basis"], dtype=np.int64),
                           pod_k=np.asarray(rows["k"], dtype=np.int64), pod_info=np.asarray(rows["info"]),
                           final_a_c=a_c, final_a_n=a_n, aggregates=aggregates)


def _run_phase(op, dts, outs, tt, wave, emit, rows, base, host_probe, device_probe, use_graph,
               record_states):
    """Run the steps dts (node times tt, output flags outs) on the device from
    the state held there; returns (a_c, a_n or None, per-step iterations,
    a_c history or None, all steps had outputs)."""
    n = len(dts)
    n_c = op.grid.n_c
    wave_tab = np.array([float(wave(x)) for x in tt])
    dt_tab = np.array(dts, dtype=np.float64)
    all_out = all(outs)
    step_iters = np.zeros((n, 4), dtype=np.int32)
    hist = np.empty((n, n_c)) if record_states else None
    failed = ctypes.c_int64(-1)
    a_n = None
    hist_n = None
    if all_out and not host_probe:
        hist_n = np.empty((n, op.grid.n_n)) if record_states else None
        rc = op.lib.mq_run_explicit_states(op.grid.ctx, n, dptr(dt_tab), dptr(wave_tab), 1,
                                           1 if use_graph else 0, _lib.i32ptr(step_iters),
                                           dptr(hist) if hist is not None else None,
                                           dptr(hist_n) if hist_n is not None else None, ctypes.byref(failed))
        if rc == _lib.MQ_NONFINITE:
            raise StepFailureError(f"non-finite conducting state at step {base + failed.value}")
        check(rc)
        a_c = op._get_state()
        blog = np.zeros(n)
        if device_probe and n > 0:
            check(op.lib.mq_run_probe_log(op.grid.ctx, n, dptr(blog)))
        # rows: one per step, window means over that step's solves
        for m in range(n):
            rows["t"].append(tt[m + 1])
            rows["b"].append(float(blog[m]))
            rows["src"].append(float(np.mean(step_iters[m, [0, 2]])))
            rows["prev"].append(float(step_iters[m, 1]))
            rows["cur"].append(float(step_iters[m, 3]))
        if n > 0:
            # per-row strategy columns from the device log (schur.py:448-467,
            # 524-538): the window of a row is one Euler step + its recovery
            dlog = np.zeros((n, 8))
            check(op.lib.mq_run_diag_log(op.grid.ctx, n, dptr(dlog)))
            if op.strategy_kind == "cspe":
                rows["basis"].extend(int(v) for v in dlog[:, 0:3].max(axis=1))
                rows["k"].extend([0] * n)
                rows["info"].extend([1.0] * n)
            elif op.strategy_kind == "pod":
                rows["basis"].extend(int(v) for v in dlog[:, 5])
                rows["k"].extend(int(v) for v in np.maximum(dlog[:, 3], dlog[:, 5]))
                rows["info"].extend(float(min(1.0, a, b)) for a, b in zip(dlog[:, 4], dlog[:, 6]))
            else:
                rows["basis"].extend([0] * n)
                rows["k"].extend([0] * n)
                rows["info"].extend([1.0] * n)
        op.solve_iterations[RhsFamily.SOURCE_CURRENT].extend(
            int(v) for pair in step_iters[:, [0, 2]] for v in pair)
        op.solve_iterations[RhsFamily.COUPLING_FROM_PREVIOUS_STATE].extend(int(v) for v in step_iters[:, 1])
        op.solve_iterations[RhsFamily.COUPLING_FROM_CURRENT_STATE].extend(int(v) for v in step_iters[:, 3])
        a_n = _final_an(op)
    else:
        win_src, win_prev, win_pod = [], [], []
        an_rows = []
        m = 0
        while m < n:
            seg = 0
            while m + seg < n and not outs[m + seg]:
                seg += 1
            seg += 1 if m + seg < n else 0
            seg = min(seg, n - m)
            it = np.zeros((seg, 2), dtype=np.int32)   # [src, cpl_prev] per step (no recovery)
            rc = op.lib.mq_run_explicit(op.grid.ctx, seg, dptr(dt_tab[m:m + seg]),
                                        dptr(wave_tab[m:m + seg + 1].copy()), 0,
                                        1 if use_graph else 0, _lib.i32ptr(it),
                                        dptr(hist[m:m + seg]) if hist is not None else None,
                                        ctypes.byref(failed))
            if rc == _lib.MQ_NONFINITE:
                raise StepFailureError(f"non-finite conducting state at step {base + m + failed.value}")
            check(rc)
            step_iters[m:m + seg, :2] = it[:, :2]
            if op.strategy_kind == "pod" and seg > 0:
                dlog = np.zeros((seg, 8))
                check(op.lib.mq_run_diag_log(op.grid.ctx, seg, dptr(dlog)))
                win_pod.extend((int(a), float(b)) for a, b in dlog[:, 3:5])
            win_src.extend(int(v) for v in it[:, 0])
            win_prev.extend(int(v) for v in it[:, 1])
            op.solve_iterations[RhsFamily.SOURCE_CURRENT].extend(int(v) for v in it[:, 0])
            op.solve_iterations[RhsFamily.COUPLING_FROM_PREVIOUS_STATE].extend(int(v) for v in it[:, 1])
            m += seg
            if outs[m - 1]:
                a_c = op._get_state()
                a_n, (r1, r2) = recover_an(op, a_c, tt[m])
                if record_states:
                    an_rows.append((m - 1, np.array(a_n)))
                step_iters[m - 1, 2:] = (r1.iterations, r2.iterations)
                emit(tt[m], a_c, a_n, win_src + [r1.iterations], win_prev, [r2.iterations], win_pod)
                win_src, win_prev, win_pod = [], [], []
        a_c = op._get_state()
        if record_states:
            hist_n = np.full((n, op.grid.n_n), np.nan)
            for row, v in an_rows:
                hist_n[row] = v
    return a_c, a_n, step_iters, (hist, hist_n) if record_states else None, all_out


TRACE_HEADER = "t,B_probe,iters_src,iters_cpl_prev,iters_cpl_cur,basis_cols,pod_k,pod_info"


def trace_bytes(result: TransientResult) -> bytes:
    """The reference's trace CSV of a transient result (bench.py:42, 341-357):
    one row per output time, floats by repr, counts as integers."""
    if result.n_rows == 0:
        raise ValueError("refusing to write an empty trace")
    out = [TRACE_HEADER]
    for i in range(result.n_rows):
        out.append(",".join([repr(float(result.times[i])), repr(float(result.probe_b[i])),
                             repr(float(result.iters_src[i])), repr(float(result.iters_cpl_prev[i])),
                             repr(float(result.iters_cpl_cur[i])), str(int(result.basis_cols[i])),
                             str(int(result.pod_k[i])), repr(float(result.pod_info[i]))]))
    return ("\n".join(out) + "\n").encode("ascii")


def _final_an(op: SchurOperator) -> np.ndarray:
    """a_n = y_src - y_cpl of the last recovery, read from the device."""
    out = np.empty(op.grid.n_n)
    check(op.lib.mq_last_an(op.grid.ctx, dptr(out)))
    return out
