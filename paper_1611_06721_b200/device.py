"""Device context: the structured FIT grid on one B200 (wraps ``mq_ctx``).

A :class:`Problem` carries what the reference's ``assemble`` consumes
(``model.py:438``): the cell material map, spacing, conductor material,
air reluctivity, plus the compact source pattern and waveform of its
``ScaledPatternSource`` (``schur.py:69-82``).  :class:`DeviceGrid` turns it
into a context holding the bit-exact partition, the active-dof bitmask and
the conducting-block index structures on the GPU.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field
from typing import Callable

import numpy as np

from . import _lib
from ._lib import check, dptr, f64, i64ptr

NU_VACUUM = 1.0 / (4e-7 * np.pi)  # model.py:63
AIR, CONDUCTOR, COIL = 0, 1, 2


@dataclass
class Problem:
    """Inputs of one magnetoquasistatic model on an nx*ny*nz cell grid."""

    material: np.ndarray                 # int8 (nx, ny, nz), C order
    h: float
    kappa: float
    brauer: tuple = (0.0, 0.0, NU_VACUUM)  # (k1, k2, k3): nu = k1 exp(k2 B^2) + k3
    nu_air: float = NU_VACUUM
    pattern: np.ndarray | None = None    # compact source pattern (n_n,)
    waveform: Callable[[float], float] | None = None
    kn_diag: float = 0.0                 # assembled K_n coefficients (0: derive)
    kn_off: float = 0.0
    name: str = ""
    meta: dict = field(default_factory=dict)

    @property
    def shape(self):
        return tuple(int(s) for s in self.material.shape)

    @classmethod
    def from_reference_model(cls, model, waveform=None) -> "Problem":
        """Adapter from a reference ``mqsolve.model.Model`` (duck-typed)."""
        grid = model.grid
        cond = model.conductor
        kn = model.system.kn
        diag = np.unique(kn.diagonal())
        rows = np.repeat(np.arange(kn.nrows), np.diff(kn.row_ptr))
        off = np.unique(np.abs(kn.values[kn.col_idx != rows]))
        if diag.size != 1 or off.size > 1:
            raise ValueError("K_n is not the constant-coefficient FIT stencil")
        src = model.system.source
        return cls(material=np.ascontiguousarray(grid.material, dtype=np.int8),
                   h=float(grid.h), kappa=float(cond.kappa),
                   brauer=(float(cond.brauer_k1), float(cond.brauer_k2),
                           float(cond.brauer_k3)),
                   nu_air=float(model.air_reluctivity),
                   pattern=np.asarray(getattr(src, "pattern", model.pattern_n), dtype=np.float64),
                   waveform=waveform or getattr(src, "waveform", None),
                   kn_diag=float(diag[0]), kn_off=float(off[0]) if off.size else 0.0)


class DeviceGrid:
    """One ``mq_ctx``: partition, masks and operators of a Problem on a GPU."""

    def __init__(self, problem: Problem, device: int = 0):
        self.lib = _lib.load()
        self.problem = problem
        mat = np.ascontiguousarray(problem.material, dtype=np.int8)
        if mat.ndim != 3:
            raise ValueError("material map must be 3-D")
        self._mat = mat
        k1, k2, k3 = problem.brauer
        desc = _lib.GridDesc(mat.shape[0], mat.shape[1], mat.shape[2], float(problem.h),
                             mat.ctypes.data_as(_lib.c_int8_p), float(problem.nu_air),
                             float(problem.kappa), float(k1), float(k2), float(k3),
                             float(problem.kn_diag), float(problem.kn_off))
        ctx = ctypes.c_void_p()
        check(self.lib.mq_ctx_create(ctypes.byref(desc), int(device), ctypes.byref(ctx)))
        self.ctx = ctx
        self.device = device
        self.n_n = int(self.lib.mq_n_n(ctx))
        self.n_c = int(self.lib.mq_n_c(ctx))
        self.dev_len = int(self.lib.mq_dev_len(ctx))
        d, o, j = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
        check(self.lib.mq_kn_coefficients(ctx, ctypes.byref(d), ctypes.byref(o), ctypes.byref(j)))
        self.kn_diag, self.kn_off, self.jacobi_inv = d.value, o.value, j.value

    # -- lifetime ------------------------------------------------------------
    def close(self):
        if getattr(self, "ctx", None):
            self.lib.mq_ctx_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- partition -------------------------------------------------------------
    def partition(self) -> tuple[np.ndarray, np.ndarray]:
        """Global edge ids of the nonconducting and conducting dofs."""
        nc = np.empty(self.n_n, dtype=np.int64)
        c = np.empty(self.n_c, dtype=np.int64)
        check(self.lib.mq_partition_export(self.ctx, i64ptr(nc), i64ptr(c)))
        return nc, c

    def noncond_index(self, global_ids) -> np.ndarray:
        g = np.ascontiguousarray(global_ids, dtype=np.int64)
        out = np.empty_like(g)
        check(self.lib.mq_map_global_to_noncond(self.ctx, i64ptr(g), g.size, i64ptr(out)))
        return out

    def pcg_kernel(self) -> tuple[str, int]:
        """(name, grid) of the fused PCG kernel this context launches."""
        buf = ctypes.create_string_buffer(64)
        grid = ctypes.c_int32()
        check(self.lib.mq_pcg_kernel_info(self.ctx, buf, 64, ctypes.byref(grid)))
        return buf.value.decode(), int(grid.value)

    def set_sm_budget(self, sms: int) -> None:
        """Confine the PCG kernel to ``sms`` SMs (0 = whole GPU)."""
        check(self.lib.mq_ctx_set_sm_budget(self.ctx, int(sms)))

    def mc_diag(self) -> np.ndarray:
        out = np.empty(self.n_c)
        check(self.lib.mq_mc_diag(self.ctx, dptr(out)))
        return out

    # -- device vectors --------------------------------------------------------
    def alloc(self) -> int:
        p = ctypes.c_void_p()
        check(self.lib.mq_vec_alloc(self.ctx, ctypes.byref(p)))
        return p.value

    def free(self, p: int):
        check(self.lib.mq_vec_free(self.ctx, ctypes.c_void_p(p)))

    def upload(self, host, dev: int):
        v = f64(host, self.n_n)
        check(self.lib.mq_vec_upload(self.ctx, dptr(v), ctypes.c_void_p(dev)))

    def download(self, dev: int) -> np.ndarray:
        out = _lib.pinned_empty(self.n_n)
        check(self.lib.mq_vec_download(self.ctx, ctypes.c_void_p(dev), dptr(out)))
        return out

    # -- operators -------------------------------------------------------------
    def kn_apply(self, x) -> np.ndarray:
        """y = K_n x (schur.py:189-191) on host compact vectors."""
        v = f64(x, self.n_n)
        y = np.empty(self.n_n)
        check(self.lib.mq_kn_apply_host(self.ctx, dptr(v), dptr(y)))
        return y

    def kc_apply(self, state, x) -> np.ndarray:
        """K_c(state) x (model.py:507-509)."""
        s = f64(state, self.n_c, "state")
        v = f64(x, self.n_c)
        y = np.empty(self.n_c)
        check(self.lib.mq_kc_apply_host(self.ctx, dptr(s), dptr(v), dptr(y)))
        return y

    def kcn_t_apply(self, a_c) -> np.ndarray:
        """K_cn^T a_c (sparse.py:187-193)."""
        v = f64(a_c, self.n_c)
        y = np.empty(self.n_n)
        check(self.lib.mq_kcn_t_apply_host(self.ctx, dptr(v), dptr(y)))
        return y

    def kcn_apply(self, x_n) -> np.ndarray:
        """K_cn x_n (sparse.py:179-184)."""
        v = f64(x_n, self.n_n)
        y = np.empty(self.n_c)
        check(self.lib.mq_kcn_apply_host(self.ctx, dptr(v), dptr(y)))
        return y

    def pcg_batched(self, b, x0=None, *, rel_tol=1e-8, abs_tol=0.0, max_iter=5000, jacobi=True):
        """nb right-hand sides (rows of ``b``, nb in 1, 2, 4, 8) of K_n in one
        member-batched launch (``mq_pcg_solve_batched_host``); returns
        (x rows, [(iterations, converged, final_rel_residual, applies)], kernel ms)."""
        b = np.ascontiguousarray(np.atleast_2d(b), dtype=np.float64)
        nb = b.shape[0]
        if b.shape[1] != self.n_n:
            raise ValueError("rhs rows must have length n_n")
        x0v = None if x0 is None else np.ascontiguousarray(np.atleast_2d(x0), dtype=np.float64)
        x = np.empty_like(b)
        reps = (_lib.SolveReportC * nb)()
        ms = ctypes.c_double()
        rc = self.lib.mq_pcg_solve_batched_host(self.ctx, nb, dptr(b), dptr(x0v) if x0v is not None else None,
                                                 dptr(x), float(rel_tol), float(abs_tol), int(max_iter),
                                                 int(bool(jacobi)), reps, ctypes.byref(ms))
        check(rc, allow=(_lib.MQ_OK, _lib.MQ_NOT_CONVERGED))
        return x, [(int(r.iterations), bool(r.converged), float(r.final_rel_residual), int(r.applies))
                   for r in reps], float(ms.value)

    def kn_operator(self) -> "KnOperator":
        return KnOperator(self)

    def sync(self):
        check(self.lib.mq_ctx_sync(self.ctx))


class KnOperator:
    """Callable ``x -> K_n x`` whose PCG runs entirely on the device.

    Mirrors the reference's counted operator (``schur.py:156-165``):
    ``count`` grows by one per application, including applications made
    inside :func:`paper_1611_06721_b200.krylov.pcg_solve`.
    """

    def __init__(self, grid: DeviceGrid):
        self.grid = grid
        self.count = 0

    @property
    def n(self) -> int:
        return self.grid.n_n

    def diagonal(self) -> np.ndarray:
        return np.full(self.grid.n_n, self.grid.kn_diag)

    def __call__(self, x):
        self.count += 1
        return self.grid.kn_apply(x)


def default_probe_cells(material) -> np.ndarray:
    """Conductor cells of the median k layer, global ids (model.py:562-566)."""
    mat = np.asarray(material)
    ijk = np.argwhere(mat == CONDUCTOR)
    if ijk.size == 0:
        raise ValueError("no conductor cells")
    mid_k = int(np.median(ijk[:, 2]))
    sel = ijk[ijk[:, 2] == mid_k]
    _, ny, nz = mat.shape
    return ((sel[:, 0] * ny + sel[:, 1]) * nz + sel[:, 2]).astype(np.int64)


def sinusoid(freq: float = 50.0) -> Callable[[float], float]:
    """Coil waveform sin(2 pi f t) of the BASELINE configs."""
    w = 2.0 * np.pi * freq
    return lambda t: math.sin(w * t)
