"""GPU ``pcg_solve``: drop-in for ``mqsolve.krylov.pcg_solve`` (krylov.py:174-250).

Same signature, stopping rule, zero-iteration shortcut, breakdown checks and
``SolveReport`` semantics as the reference; the whole solve is one persistent
cooperative kernel on the device.  Operators:

* :class:`~paper_1611_06721_b200.device.KnOperator` — the matrix-free K_n
  stencil of a :class:`DeviceGrid` (the hot path), scalar Jacobi;
* a CsrMatrix-like object (``row_ptr``/``col_idx``/``values``), a scipy
  sparse matrix or a square ndarray — the general CSR kernel path.

Python callables cannot run on the device and raise ``TypeError``.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from enum import Enum

import numpy as np

from . import _lib
from ._lib import check, dptr, f64

__all__ = ["Preconditioner", "PcgConfig", "SolveReport", "JacobiPreconditioner",
           "IndefiniteOperatorError", "pcg_solve"]


class Preconditioner(str, Enum):
    NONE = "none"
    JACOBI = "jacobi"
    IC0 = "ic0"


class IndefiniteOperatorError(RuntimeError):
    """A CG search direction exposed an indefinite operator (krylov.py:44-45)."""


@dataclass(frozen=True)
class PcgConfig:
    """krylov.py:57-72."""

    rel_tol: float = 1e-8
    abs_tol: float = 0.0
    max_iter: int = 5000
    preconditioner: Preconditioner = Preconditioner.NONE

    def __post_init__(self):
        if not (self.rel_tol > 0.0):
            raise ValueError("rel_tol must be positive")
        if self.abs_tol < 0.0:
            raise ValueError("abs_tol must be nonnegative")
        if self.max_iter < 1:
            raise ValueError("max_iter must be at least 1")
        object.__setattr__(self, "preconditioner", Preconditioner(self.preconditioner))


@dataclass(frozen=True)
class SolveReport:
    """krylov.py:75-79, plus the operator applications the device counted."""

    iterations: int
    final_rel_residual: float
    converged: bool
    applications: int = 0


class JacobiPreconditioner:
    """M^-1 = diag(1/A_ii), identity on zero entries (krylov.py:82-97)."""

    def __init__(self, diag):
        d = f64(diag, name="diagonal")
        if (d < 0).any():
            raise ValueError("Jacobi preconditioner requires a nonnegative diagonal")
        self._inv = np.where(d > 0, 1.0 / np.where(d > 0, d, 1.0), 1.0)

    @property
    def inverse(self) -> np.ndarray:
        return self._inv

    def apply(self, r):
        return self._inv * r


def _inverse_of(pre, n):
    """Diagonal of a Jacobi-type preconditioner object, or raise."""
    inv = getattr(pre, "_inv", None)
    if inv is None:
        raise NotImplementedError(
            f"{type(pre).__name__} has no device implementation (Jacobi only)")
    inv = np.ascontiguousarray(inv, dtype=np.float64)
    if inv.shape != (n,):
        raise ValueError("preconditioner size mismatch")
    return inv


def _csr_of(a):
    """(n, row_ptr int64, col_idx int32, values) of a matrix operator."""
    import scipy.sparse as sp
    if hasattr(a, "row_ptr") and hasattr(a, "col_idx") and hasattr(a, "values"):
        if a.nrows != a.ncols:
            raise ValueError("operator must be square")
        return (int(a.nrows), np.ascontiguousarray(a.row_ptr, dtype=np.int64),
                np.ascontiguousarray(a.col_idx, dtype=np.int32),
                np.ascontiguousarray(a.values, dtype=np.float64))
    if sp.issparse(a):
        m = sp.csr_matrix(a)
        if m.shape[0] != m.shape[1]:
            raise ValueError("operator must be square")
        m.sort_indices()
        return (m.shape[0], m.indptr.astype(np.int64), m.indices.astype(np.int32),
                m.data.astype(np.float64))
    if isinstance(a, np.ndarray):
        if a.ndim != 2 or a.shape[0] != a.shape[1]:
            raise ValueError("dense operator must be square")
        m = sp.csr_matrix(np.asarray(a, dtype=np.float64))
        m.sort_indices()
        return (m.shape[0], m.indptr.astype(np.int64), m.indices.astype(np.int32),
                m.data.astype(np.float64))
    return None


def pcg_solve(a, b, x0=None, config: PcgConfig | None = None, preconditioner=None,
              device: int = 0):
    """Solve A x = b by preconditioned CG on the GPU (krylov.py:174-250).

    Returns ``(x, SolveReport)``; ``converged=False`` with the last iterate
    when the budget is exhausted; indefiniteness raises
    :class:`IndefiniteOperatorError`.
    """
    from .device import KnOperator
    config = config or PcgConfig()
    lib = _lib.load()
    rep = _lib.SolveReportC()
    if isinstance(a, KnOperator):
        g = a.grid
        bv = f64(b, g.n_n, "rhs")
        if not np.isfinite(bv).all():
            raise ValueError("rhs contains non-finite entries")
        x0v = None
        if x0 is not None:
            x0v = f64(x0, g.n_n, "start vector")
            if not np.isfinite(x0v).all():
                raise ValueError("start vector contains non-finite entries")
        use_jac = 0
        if preconditioner is not None:
            inv = _inverse_of(preconditioner, g.n_n)
            if not np.all(inv == g.jacobi_inv):
                raise NotImplementedError("K_n stencil path supports its own Jacobi only")
            use_jac = 1
        elif config.preconditioner is Preconditioner.JACOBI:
            use_jac = 1
        elif config.preconditioner is Preconditioner.IC0:
            raise NotImplementedError("IC(0) is not part of the device path")
        x = np.empty(g.n_n)
        rc = lib.mq_pcg_solve_host(g.ctx, dptr(bv), dptr(x0v) if x0v is not None else None,
                                   dptr(x), config.rel_tol, config.abs_tol, config.max_iter,
                                   use_jac, ctypes.byref(rep))
        check(rc, allow=(_lib.MQ_OK, _lib.MQ_NOT_CONVERGED))
        a.count += int(rep.applies)
        return x, SolveReport(int(rep.iterations), float(rep.final_rel_residual),
                              bool(rep.converged), int(rep.applies))
    from .csrsys import CsrOperator
    if isinstance(a, CsrOperator):
        # a block resident on the device (models given as matrices)
        use_jac = config.preconditioner is Preconditioner.JACOBI
        if preconditioner is not None:
            inv = _inverse_of(preconditioner, a.n)
            if a.inverse is None or not np.array_equal(inv, a.inverse):
                raise NotImplementedError("a resident CSR block solves with its own Jacobi inverse only")
            use_jac = True
        elif config.preconditioner is Preconditioner.IC0:
            raise NotImplementedError("IC(0) is not part of the device path")
        return a.solve(b, x0=x0, config=config, use_jacobi=use_jac)
    csr = _csr_of(a)
    if csr is None:
        if callable(a):
            raise TypeError("the device PCG needs a matrix or a DeviceGrid K_n operator, "
                            "not an arbitrary Python callable")
        raise TypeError(f"unsupported operator type {type(a).__name__}")
    n, rp, ci, va = csr
    bv = f64(b, n, "rhs")
    if not np.isfinite(bv).all():
        raise ValueError("rhs contains non-finite entries")
    x0v = None
    if x0 is not None:
        x0v = f64(x0, n, "start vector")
        if not np.isfinite(x0v).all():
            raise ValueError("start vector contains non-finite entries")
    inv = None
    if preconditioner is not None:
        inv = _inverse_of(preconditioner, n)
    elif config.preconditioner is Preconditioner.JACOBI:
        inv = JacobiPreconditioner(_diag_of(n, rp, ci, va)).inverse
    elif config.preconditioner is Preconditioner.IC0:
        raise NotImplementedError("IC(0) is not part of the device path")
    x = np.zeros(n)
    rc = lib.mq_csr_pcg_solve(device, n, _lib.i64ptr(rp), _lib.i32ptr(ci), dptr(va), dptr(bv),
                              dptr(x0v) if x0v is not None else None, dptr(x),
                              dptr(inv) if inv is not None else None, config.rel_tol,
                              config.abs_tol, config.max_iter, ctypes.byref(rep))
    check(rc, allow=(_lib.MQ_OK, _lib.MQ_NOT_CONVERGED))
    if hasattr(a, "count"):
        a.count += int(rep.applies)
    return x, SolveReport(int(rep.iterations), float(rep.final_rel_residual),
                          bool(rep.converged), int(rep.applies))


def _diag_of(n, rp, ci, va):
    d = np.zeros(n)
    rows = np.repeat(np.arange(n), np.diff(rp))
    on = ci == rows
    d[rows[on]] = va[on]
    return d


def csr_spmv(a, x, device: int = 0) -> np.ndarray:
    """y = A x for a CSR-like matrix on the device (sparse.py:179-184)."""
    n, rp, ci, va = _csr_of(a)
    ncols = int(getattr(a, "ncols", n))
    xv = f64(x, ncols)
    y = np.empty(n)
    check(_lib.load().mq_csr_spmv(device, n, ncols, _lib.i64ptr(rp), _lib.i32ptr(ci), dptr(va),
                                  dptr(xv), dptr(y)))
    return y
