"""Device start-vector strategies (drop-in for ``mqsolve.startvec``).

:class:`DeviceStrategy` implements the reference's ``StartVectorStrategy``
protocol (startvec.py:315-342: ``kind``, ``start_vector``, ``observe``,
``basis_size``, ``maintenance_applies``, ``diagnostics``) with the CSPE
cache (startvec.py:118-225), the POD snapshot projection
(startvec.py:239-309) or the previous-solution rule (startvec.py:345-359)
running on the GPU against the matrix-free K_n of a :class:`DeviceGrid`.
An instance can be injected into the reference's ``SchurOperator`` through
``strategy=`` (schur.py:198-199); its operator argument is not needed
because K_n lives on the device.
"""

from __future__ import annotations

import ctypes
from enum import Enum

import numpy as np

from . import _lib
from ._lib import check, dptr, f64

__all__ = ["RhsFamily", "DeviceStrategy", "FAMILY_INDEX"]


class RhsFamily(Enum):
    """startvec.py:45-50."""

    SOURCE_CURRENT = "source"
    COUPLING_FROM_CURRENT_STATE = "coupling_current"
    COUPLING_FROM_PREVIOUS_STATE = "coupling_previous"


FAMILY_INDEX = {"source": _lib.FAM_SOURCE, "coupling_current": _lib.FAM_COUPLING_CURRENT,
                "coupling_previous": _lib.FAM_COUPLING_PREVIOUS}


def family_index(family) -> int:
    val = getattr(family, "value", family)
    return FAMILY_INDEX[str(val)]


def solver_cfg(kind: str, *, max_cols=20, n_pod=10, eps_pod=1e-4, rel_tol=1e-8,
               abs_tol=0.0, max_iter=5000, drop_tol=None) -> _lib.SolverCfg:
    kind = str(kind).lower()
    if kind not in _lib.STRAT:
        raise ValueError(f"unknown start-vector strategy {kind!r}")
    return _lib.SolverCfg(_lib.STRAT[kind], int(max_cols), int(n_pod), int(max_iter),
                          float(eps_pod), float(rel_tol), float(abs_tol),
                          float(rel_tol if drop_tol is None else drop_tol))


class DeviceStrategy:
    """StartVectorStrategy protocol backed by the device solver of a grid."""

    def __init__(self, grid, kind="cspe", *, max_cols=20, n_pod=10, eps_pod=1e-4,
                 drop_tol=1e-10):
        self.grid = grid
        self.kind = str(kind).lower()
        self.dim = grid.n_n
        self.max_cols, self.n_pod, self.eps_pod = max_cols, n_pod, eps_pod
        cfg = solver_cfg(self.kind, max_cols=max_cols, n_pod=n_pod, eps_pod=eps_pod,
                         drop_tol=drop_tol)
        check(grid.lib.mq_solver_init(grid.ctx, ctypes.byref(cfg), None))
        self._rhs = grid.alloc()
        self._x0 = grid.alloc()
        self._y = grid.alloc()
        self._basis_sizes = [0, 0, 0]

    def start_vector(self, family, rhs) -> np.ndarray:
        fam = family_index(family)
        if rhs is None:
            rhs = np.zeros(self.dim)
        self.grid.upload(f64(rhs, self.dim, "rhs"), self._rhs)
        check(self.grid.lib.mq_strategy_start(self.grid.ctx, fam, ctypes.c_void_p(self._rhs),
                                              ctypes.c_void_p(self._x0)))
        return self.grid.download(self._x0)

    def observe(self, family, solution) -> None:
        fam = family_index(family)
        self.grid.upload(f64(solution, self.dim, "solution"), self._y)
        check(self.grid.lib.mq_strategy_observe(self.grid.ctx, fam, ctypes.c_void_p(self._y)))

    def _diag(self) -> _lib.Diag:
        d = _lib.Diag()
        check(self.grid.lib.mq_diagnostics(self.grid.ctx, ctypes.byref(d)))
        return d

    def basis_size(self, family=None) -> int:
        d = self._diag()
        if self.kind == "pod":
            return int(d.pod_k)
        if self.kind != "cspe":
            return 0
        if family is not None:
            return int(d.basis_cols[family_index(family)])
        return int(max(d.basis_cols))

    @property
    def maintenance_applies(self) -> int:
        return int(self._diag().maintenance_applies)

    def diagnostics(self) -> dict:
        d = self._diag()
        if self.kind == "cspe":
            return {"basis_cols": int(max(d.basis_cols)),
                    "maintenance_applies": int(d.maintenance_applies)}
        if self.kind == "pod":
            return {"pod_k": int(d.pod_k), "pod_info": float(d.pod_info),
                    "min_pod_info": float(d.min_pod_info),
                    "maintenance_applies": int(d.maintenance_applies)}
        return {}

    def cache_export(self, family):
        """(basis U, cached products K U, Galerkin U^T K U) of one CSPE family."""
        fam = family_index(family)
        k = ctypes.c_int32()
        n = self.dim
        U = np.empty((32, n))
        KU = np.empty((32, n))
        G = np.empty(32 * 32)
        check(self.grid.lib.mq_cspe_export(self.grid.ctx, fam, ctypes.byref(k), dptr(U),
                                           dptr(KU), dptr(G)))
        kk = k.value
        return U[:kk].T.copy(), KU[:kk].T.copy(), G[:kk * kk].reshape(kk, kk).copy()
