"""Models given as matrices (the reference's manifest path) on the GPU.

``mqsolve``'s ``load_model`` (bench.py:228-313) turns an ``export_model``
directory (model.py:640-689: five Matrix Market blocks and ``manifest.json``)
into a ``PartitionedSystem`` of CSR blocks with no grid behind it, so the
stencil kernels do not apply.  Here:

* :func:`load_manifest` reads such a directory with the reference's checks and
  returns a :class:`CsrSystem`; besides the reference's ``exponential_ramp``
  waveform it accepts ``{"kind": "sinusoid", "frequency": f}`` (the
  BASELINE configs' coil current);
* :class:`CsrOperator` keeps one block resident on the device (C ABI
  ``mq_csr_op_*``); :func:`pcg_solve` takes it like a ``KnOperator`` and the
  call counts its applications like ``_CountedApply`` (schur.py:189-191);
* :class:`CsrSchurOperator` with :func:`explicit_euler_step`,
  :func:`recover_an` and :func:`run_explicit` steps the frozen-linear system
  (schur.py:239-264, 379-419, 474-607) with every K_n solve on the device and
  the K_cn / K_c products as device SpMVs.  Start vectors: ``"zero"``,
  ``"previous"`` or any ``StartVectorStrategy`` object (startvec.py:315-342,
  e.g. the reference's own ``CspeStrategy`` for these models).
"""

from __future__ import annotations

import ctypes
import json
import math
from dataclasses import dataclass, field
from pathlib import Path
from typing import Callable

import numpy as np

from . import _lib
from ._lib import check, dptr
from .krylov import JacobiPreconditioner, PcgConfig, Preconditioner, SolveReport
from .startvec import RhsFamily


class ConfigError(ValueError):
    """bench.py's ConfigError: a manifest that cannot be loaded."""


BLOCKS = ("m_c", "k_c", "k_cn", "k_n", "source_pattern")


def _csr_arrays(m):
    """CsrMatrix.from_scipy (sparse.py:118-122): duplicates summed, column
    indices sorted per row; int64 row pointers, int32 columns."""
    import scipy.sparse as sp
    c = sp.csr_matrix(m, dtype=np.float64)
    c.sum_duplicates()
    c.sort_indices()
    return c


def read_matrix_market(path):
    """sparse.py:224-229 (symmetric storage expands to full)."""
    import scipy.io
    m = scipy.io.mmread(str(path))
    return _csr_arrays(m)


def read_dense_vector(path) -> np.ndarray:
    """sparse.py:241-247."""
    import scipy.io
    m = scipy.io.mmread(str(path))
    if not isinstance(m, np.ndarray):
        m = m.toarray()
    if m.ndim != 2 or 1 not in m.shape:
        raise ValueError(f"{path} does not hold a single vector")
    v = np.ascontiguousarray(m.ravel(), dtype=np.float64)
    if not np.isfinite(v).all():
        raise ValueError(f"{path} contains non-finite entries")
    return v


def exponential_ramp(tau: float) -> Callable[[float], float]:
    """schur.py:62-66."""
    if tau <= 0:
        raise ValueError("tau must be positive")
    return lambda t: 1.0 - np.exp(-t / tau)


def sinusoid_waveform(frequency: float, amplitude: float = 1.0) -> Callable[[float], float]:
    """amplitude * sin(2 pi f t) (the BASELINE configs' coil current)."""
    if not frequency > 0:
        raise ValueError("frequency must be positive")
    w = 2.0 * math.pi * frequency
    return lambda t: amplitude * math.sin(w * t)


def _symmetric(c, tol) -> bool:
    d = abs(c - c.T)
    return d.nnz == 0 or float(d.max()) <= tol


@dataclass
class CsrSystem:
    """The frozen-linear PartitionedSystem of a manifest (schur.py:85-160):
    conducting mass (diagonal used, schur.py:212), K_c at the zero state,
    K_cn, K_n (scipy CSR, CsrMatrix order) and the source pattern x waveform."""

    mc: object
    kc: object
    kcn: object
    kn: object
    pattern: np.ndarray
    waveform: Callable[[float], float]
    manifest: dict = field(default_factory=dict)
    builtin: object = None   # Problem rebuilt from the manifest's "builtin" section (FIT grid)

    @property
    def n_c(self) -> int:
        return int(self.kcn.shape[0])

    @property
    def n_n(self) -> int:
        return int(self.kcn.shape[1])

    def validate(self) -> None:
        """PartitionedSystem.validate (schur.py:113-143): shapes, positive
        conducting mass diagonal."""
        n_c, n_n = self.n_c, self.n_n
        for name, blk, shape in (("m_c", self.mc, (n_c, n_c)), ("k_c", self.kc, (n_c, n_c)),
                                 ("k_n", self.kn, (n_n, n_n))):
            if blk.shape != shape:
                raise ConfigError(f"block {name!r} has shape {blk.shape}, expected {shape}")
        if self.pattern.size != n_n:
            raise ConfigError(f"block 'source_pattern' has length {self.pattern.size}, expected {n_n}")
        if not np.all(self.mc.diagonal() > 0):
            raise ConfigError("conducting mass diagonal must be positive")


def _require(d, key, where):
    if not isinstance(d, dict) or key not in d:
        raise ConfigError(f"{where} lacks {key!r}")
    return d[key]


def load_manifest(path) -> CsrSystem:
    """bench.py:228-313 for the stored blocks (a frozen-linear system).

    A ``builtin`` section (bench.py:283-306: the reference rebuilds its FIT
    model from it and refuses stored blocks that disagree) rebuilds the model
    as a :class:`~paper_1611_06721_b200.device.Problem` in ``system.builtin``
    (configs.builtin_problem) — the stencil path, which also carries the
    Brauer nonlinearity — and checks the stored source pattern against it
    here; the stored matrix blocks are checked against the rebuilt model on
    the device when a :class:`CsrSchurOperator` is made (verify_builtin),
    which also refuses to step a nonlinear builtin model as frozen-linear."""
    path = Path(path)
    mpath = path / "manifest.json" if path.is_dir() else path
    if not mpath.exists():
        raise ConfigError(f"manifest not found: {mpath}")
    try:
        manifest = json.loads(mpath.read_text())
    except json.JSONDecodeError as err:
        raise ConfigError(f"manifest is not valid JSON: {err}")
    if manifest.get("format") != "mqsolve-model":
        raise ConfigError("manifest format marker missing or unknown")
    blocks = _require(manifest, "blocks", "manifest")
    loaded = {}
    for name in BLOCKS:
        entry = _require(blocks, name, "manifest blocks section")
        fp = mpath.parent / _require(entry, "file", f"block {name!r}")
        if not fp.exists():
            raise ConfigError(f"block {name!r} file not found: {fp}")
        loaded[name] = read_dense_vector(fp) if name == "source_pattern" else read_matrix_market(fp)
    for name in ("k_c", "k_n"):
        blk = loaded[name]
        scale = float(np.abs(blk.data).max()) if blk.nnz else 1.0
        if not _symmetric(blk, 1e-12 * scale):
            raise ConfigError(f"block {name!r} is asymmetric beyond a relative tolerance of 1e-12")
    wf = _require(manifest, "waveform", "manifest")
    kind = wf.get("kind")
    if kind == "exponential_ramp":
        waveform = exponential_ramp(float(_require(wf, "tau", "waveform section")))
    elif kind == "sinusoid":
        waveform = sinusoid_waveform(float(_require(wf, "frequency", "waveform section")),
                                     float(wf.get("amplitude", 1.0)))
    else:
        raise ConfigError(f"unknown waveform kind {kind!r}")
    system = CsrSystem(mc=loaded["m_c"], kc=loaded["k_c"], kcn=loaded["k_cn"], kn=loaded["k_n"],
                       pattern=loaded["source_pattern"], waveform=waveform, manifest=manifest)
    builtin = manifest.get("builtin")
    if builtin:
        from .configs import builtin_problem
        try:
            prob = builtin_problem(cells=int(builtin["cells"]), h=float(builtin["h"]),
                                   kappa=float(builtin["kappa"]), brauer=tuple(builtin["brauer"]),
                                   amps=float(builtin["amps"]), tau=float(builtin["tau"]),
                                   linear=bool(builtin["linear"]))
        except (KeyError, TypeError, ValueError) as err:
            raise ConfigError(f"builtin section cannot be rebuilt: {err}")
        if prob.pattern.shape != system.pattern.shape or not np.array_equal(prob.pattern, system.pattern):
            raise ConfigError("stored source pattern disagrees with the builtin parameters in the manifest")
        system.builtin = prob
        system.waveform = prob.waveform
    system.validate()
    return system


def is_diagonal(m) -> bool:
    """CsrMatrix.is_diagonal (sparse.py:166-173)."""
    c = _csr_arrays(m)
    if c.shape[0] != c.shape[1]:
        return False
    counts = np.diff(c.indptr)
    if (counts > 1).any():
        return False
    rows = np.repeat(np.arange(c.shape[0]), counts)
    return bool((c.indices == rows).all())


def _close(a, b, tol) -> bool:
    nb = float(np.linalg.norm(b))
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b))) <= tol * (nb if nb > 0 else 1.0)


def verify_builtin(system: CsrSystem, device: int = 0, seed: int = 0) -> None:
    """bench.py:291-306 on the device: the stored M_c, K_c(0), K_cn and K_n
    must be the rebuilt builtin model's blocks.  Compared through their
    products with random vectors, which the device forms in the reference's
    summation order (bit-exact for M_c, K_cn, K_cn^T, K_n; K_c to 1e-12, see
    below), so any stored entry that differs shows."""
    from .device import DeviceGrid
    prob = system.builtin
    if prob is None:
        return
    rng = np.random.default_rng(seed)
    with DeviceGrid(prob, device) as g:
        if (g.n_c, g.n_n) != (system.n_c, system.n_n):
            raise ConfigError("stored block 'k_cn' disagrees with the builtin parameters in the manifest")
        xn = rng.standard_normal(g.n_n)
        xc = rng.standard_normal(g.n_c)
        checks = (("m_c", is_diagonal(system.mc) and np.array_equal(system.mc.diagonal(), g.mc_diag())),
                  # the device forms K_c x as the reference's kc_apply closure
                  # (C^T diag(w/h) C x, model.py:507-509), not as the assembled
                  # matrix's rows: equal to rounding, not bitwise
                  ("k_c", _close(system.kc @ xc, g.kc_apply(np.zeros(g.n_c), xc), 1e-12)),
                  ("k_cn", np.array_equal(system.kcn @ xn, g.kcn_apply(xn))
                   and np.array_equal(system.kcn.T @ xc, g.kcn_t_apply(xc))),
                  ("k_n", np.array_equal(system.kn @ xn, g.kn_apply(xn))))
        for name, ok in checks:
            if not ok:
                raise ConfigError(f"stored block {name!r} disagrees with the builtin parameters in the manifest")


class CsrOperator:
    """A CSR block resident on the device.  ``op(x)`` is ``A @ x`` (counted,
    schur.py:189-191); :func:`pcg_solve` accepts it; the Jacobi inverse
    1/diag (krylov.py:90-94) is uploaded with a square block."""

    def __init__(self, matrix, device: int = 0, jacobi: bool | None = None):
        c = _csr_arrays(matrix)
        self.shape = c.shape
        self.n = int(c.shape[0])
        self.count = 0
        self.lib = _lib.load()
        rp = np.ascontiguousarray(c.indptr, dtype=np.int64)
        ci = np.ascontiguousarray(c.indices, dtype=np.int32)
        va = np.ascontiguousarray(c.data, dtype=np.float64)
        square = c.shape[0] == c.shape[1]
        self.inverse = None
        if (jacobi if jacobi is not None else square) and square:
            self.inverse = np.ascontiguousarray(JacobiPreconditioner(c.diagonal()).inverse)
        self.op = ctypes.c_void_p()
        check(self.lib.mq_csr_op_create(int(device), c.shape[0], c.shape[1], _lib.i64ptr(rp), _lib.i32ptr(ci),
                                        dptr(va), dptr(self.inverse) if self.inverse is not None else None,
                                        ctypes.byref(self.op)))

    def __call__(self, x) -> np.ndarray:
        xv = np.ascontiguousarray(x, dtype=np.float64)
        if xv.shape != (self.shape[1],):
            raise ValueError(f"vector of length {self.shape[1]} expected")
        y = np.empty(self.shape[0])
        check(self.lib.mq_csr_op_spmv(self.op, dptr(xv), dptr(y)))
        self.count += 1
        return y

    def solve(self, b, x0=None, config: PcgConfig | None = None, use_jacobi: bool = True):
        """pcg_solve on the resident block (krylov.py:174-250)."""
        config = config or PcgConfig()
        bv = np.ascontiguousarray(b, dtype=np.float64)
        if bv.shape != (self.n,):
            raise ValueError(f"rhs must be a vector of length {self.n}")
        if not np.isfinite(bv).all():
            raise ValueError("rhs contains non-finite entries")
        x0v = None
        if x0 is not None:
            x0v = np.ascontiguousarray(x0, dtype=np.float64)
            if x0v.shape != (self.n,):
                raise ValueError(f"start vector must have length {self.n}")
            if not np.isfinite(x0v).all():
                raise ValueError("start vector contains non-finite entries")
        x = np.empty(self.n)
        rep = _lib.SolveReportC()
        rc = self.lib.mq_csr_op_pcg(self.op, dptr(bv), dptr(x0v) if x0v is not None else None, dptr(x),
                                    1 if use_jacobi else 0, config.rel_tol, config.abs_tol, config.max_iter,
                                    ctypes.byref(rep))
        check(rc, allow=(_lib.MQ_OK, _lib.MQ_NOT_CONVERGED))
        self.count += int(rep.applies)
        return x, SolveReport(int(rep.iterations), float(rep.final_rel_residual), bool(rep.converged),
                              int(rep.applies))

    def close(self) -> None:
        if self.op:
            self.lib.mq_csr_op_destroy(self.op)
            self.op = ctypes.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class _ZeroStrategy:
    kind = "zero"

    def __init__(self, n):
        self.n = n

    def start_vector(self, family, rhs):
        return np.zeros(self.n)

    def observe(self, family, solution):
        pass

    def basis_size(self, family=None):
        return 0

    maintenance_applies = 0

    def diagnostics(self):
        return {"basis_cols": 0, "pod_k": 0, "pod_info": 1.0, "min_pod_info": 1.0, "maintenance_applies": 0}


class _PreviousStrategy(_ZeroStrategy):
    """startvec.py:345-359."""

    kind = "previous"

    def __init__(self, n):
        super().__init__(n)
        self.last = {}

    def start_vector(self, family, rhs):
        v = self.last.get(family)
        return np.zeros(self.n) if v is None else v.copy()

    def observe(self, family, solution):
        self.last[family] = np.array(solution, dtype=np.float64)


class StepFailureError(RuntimeError):
    """schur.py's StepFailureError."""


class CsrSchurOperator:
    """SchurOperator (schur.py:168-313) over a :class:`CsrSystem`: K_n, K_cn,
    K_cn^T and K_c resident on the device."""

    def __init__(self, system: CsrSystem, pcg: PcgConfig | None = None, strategy="previous",
                 device: int = 0, preconditioner=Preconditioner.JACOBI):
        system.validate()
        if system.builtin is not None:
            verify_builtin(system, device)
            if not system.builtin.meta.get("linear", False):
                raise ConfigError("the manifest's builtin model is nonlinear (Brauer K_c); its blocks hold K_c "
                                  "at the zero state only: step it on the stencil path, "
                                  "SchurOperator(system.builtin)")
        pre = Preconditioner(preconditioner)
        if pre is Preconditioner.IC0:
            raise NotImplementedError("IC(0) is not part of the device path (the reference falls back to "
                                      "Jacobi when it breaks down on the singular block)")
        self.use_jacobi = pre is Preconditioner.JACOBI   # schur.py:193-197
        self.system = system
        self.pcg = pcg or PcgConfig()
        self.kn = CsrOperator(system.kn, device)
        self.kcn = CsrOperator(system.kcn, device, jacobi=False)
        self.kcn_t = CsrOperator(system.kcn.T, device, jacobi=False)
        self.kc = CsrOperator(system.kc, device, jacobi=False)
        # schur.py:210-218: 1/diag for a diagonal M_c, else a Jacobi-PCG mass solve
        if is_diagonal(system.mc):
            self.minv_diag = 1.0 / system.mc.diagonal()
            self.mc = None
        else:
            self.minv_diag = None
            self.mc = CsrOperator(system.mc, device)
        n = system.n_n
        if isinstance(strategy, str):
            s = strategy.lower()
            if s == "zero":
                strategy = _ZeroStrategy(n)
            elif s == "previous":
                strategy = _PreviousStrategy(n)
            else:
                raise ValueError("CSR systems take 'zero', 'previous' or a StartVectorStrategy object")
        self.strategy = strategy
        self.solve_iterations = {f: [] for f in RhsFamily}
        self.pcg_applies = 0

    def solve_kn(self, rhs, family: RhsFamily):
        """schur.py:239-264."""
        x0 = self.strategy.start_vector(family, rhs)
        y, rep = self.kn.solve(rhs, x0=x0, config=self.pcg, use_jacobi=self.use_jacobi)
        if not rep.converged:
            raise StepFailureError(f"K_n solve ({family.value}) did not converge: "
                                   f"rel. residual {rep.final_rel_residual:.3e}")
        self.pcg_applies += rep.applications
        self.strategy.observe(family, y)
        self.solve_iterations[family].append(rep.iterations)
        return y, rep

    def source_solution(self, t: float):
        """schur.py:266-278."""
        return self.solve_kn(self.system.pattern * float(self.system.waveform(t)), RhsFamily.SOURCE_CURRENT)

    def minv(self, x) -> np.ndarray:
        """schur.py:280-287."""
        if self.minv_diag is not None:
            return self.minv_diag * x
        y, rep = self.mc.solve(np.ascontiguousarray(x, dtype=np.float64), config=self.pcg, use_jacobi=True)
        if not rep.converged:
            raise StepFailureError("conductivity mass solve stalled")
        return y

    def close(self):
        for op in (self.kn, self.kcn, self.kcn_t, self.kc) + ((self.mc,) if self.mc is not None else ()):
            op.close()


def explicit_euler_step(state, dt: float, op: CsrSchurOperator, step_index: int | None = None):
    """schur.py:379-405 on the frozen-linear CSR system."""
    a_c, t = state
    if dt < 0:
        raise ValueError("dt must be nonnegative")
    a_c = np.ascontiguousarray(a_c, dtype=np.float64)
    t_new = t + dt
    y_src, r1 = op.source_solution(t_new)
    y_cpl, r2 = op.solve_kn(op.kcn_t(a_c), RhsFamily.COUPLING_FROM_PREVIOUS_STATE)
    rate = op.kcn(y_cpl - y_src) - op.kc(a_c)
    a_next = a_c + dt * op.minv(rate)
    if not np.isfinite(a_next).all():
        where = f" at step {step_index}" if step_index is not None else ""
        raise StepFailureError(f"non-finite conducting state{where} (t = {t_new:.6e})")
    return a_next, (r1, r2)


def recover_an(op: CsrSchurOperator, a_c, t: float):
    """schur.py:408-419."""
    a_c = np.ascontiguousarray(a_c, dtype=np.float64)
    y_src, r1 = op.source_solution(t)
    y_cpl, r2 = op.solve_kn(op.kcn_t(a_c), RhsFamily.COUPLING_FROM_CURRENT_STATE)
    return y_src - y_cpl, (r1, r2)


@dataclass
class CsrTransient:
    """The TransientResult fields a CSR system produces (schur.py:422-443)."""

    times: np.ndarray
    iters_src: np.ndarray
    iters_cpl_prev: np.ndarray
    iters_cpl_cur: np.ndarray
    final_a_c: np.ndarray
    final_a_n: np.ndarray | None
    a_c_history: list = field(default_factory=list)
    pcg_applies: int = 0


def run_explicit(system: CsrSystem, t_end: float, dt: float, *, strategy="previous",
                 pcg: PcgConfig | None = None, output_period: float | None = None, a0=None,
                 device: int = 0, record_states: bool = False) -> CsrTransient:
    """schur.py:474-607 with a fixed dt: the reference's step sizes and output
    rows (schur.py:546-572); a_n recovered at every output row."""
    from .schur import step_times
    op = CsrSchurOperator(system, pcg=pcg, strategy=strategy, device=device)
    try:
        period = output_period if output_period is not None else t_end
        dts, outs = step_times(t_end, dt, period)
        a = np.zeros(system.n_c) if a0 is None else np.array(a0, dtype=np.float64)
        t = 0.0
        times, it_s, it_p, it_c, hist = [0.0], [], [], [], []
        a_n, _ = recover_an(op, a, t)
        for k, (h, out) in enumerate(zip(dts, outs)):
            a, (r1, r2) = explicit_euler_step((a, t), h, op, k + 1)
            t += h
            it_s.append(r1.iterations)
            it_p.append(r2.iterations)
            if record_states:
                hist.append(a.copy())
            if out:
                a_n, (_, q2) = recover_an(op, a, t)
                it_c.append(q2.iterations)
                times.append(t)
        return CsrTransient(times=np.array(times), iters_src=np.array(it_s), iters_cpl_prev=np.array(it_p),
                            iters_cpl_cur=np.array(it_c), final_a_c=a, final_a_n=a_n, a_c_history=hist,
                            pcg_applies=op.pcg_applies)
    finally:
        op.close()
