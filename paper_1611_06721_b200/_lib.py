"""ctypes binding of ``libmq_b200.so`` (C ABI declared in ``include/mq_b200.h``).

There is no fallback: if the shared library is missing or no CUDA device is
visible, the calls raise.  Build the library with
``python -c "import __graft_entry__ as g; g.build()"`` or
``python -m paper_1611_06721_b200.build``.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

LIB_NAME = "libmq_b200.so"
LIB_PATH = Path(__file__).resolve().parent / LIB_NAME

MQ_OK = 0
MQ_NOT_CONVERGED = 1
MQ_INDEFINITE = 2
MQ_INVALID = 3
MQ_CUDA_ERROR = 4
MQ_NONFINITE = 5

FAM_SOURCE = 0
FAM_COUPLING_CURRENT = 1
FAM_COUPLING_PREVIOUS = 2

STRAT = {"zero": 0, "previous": 1, "cspe": 2, "pod": 3}

c_double_p = ctypes.POINTER(ctypes.c_double)
c_int64_p = ctypes.POINTER(ctypes.c_int64)
c_int32_p = ctypes.POINTER(ctypes.c_int32)
c_int8_p = ctypes.POINTER(ctypes.c_int8)


class GridDesc(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int32), ("ny", ctypes.c_int32), ("nz", ctypes.c_int32),
                ("h", ctypes.c_double), ("material", c_int8_p),
                ("nu_air", ctypes.c_double), ("kappa", ctypes.c_double),
                ("brauer_k1", ctypes.c_double), ("brauer_k2", ctypes.c_double),
                ("brauer_k3", ctypes.c_double), ("kn_diag", ctypes.c_double),
                ("kn_off", ctypes.c_double)]


class SolveReportC(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int32), ("converged", ctypes.c_int32),
                ("final_rel_residual", ctypes.c_double), ("applies", ctypes.c_int64)]


class SolverCfg(ctypes.Structure):
    _fields_ = [("strategy", ctypes.c_int32), ("max_cols", ctypes.c_int32),
                ("n_pod", ctypes.c_int32), ("max_iter", ctypes.c_int32),
                ("eps_pod", ctypes.c_double), ("rel_tol", ctypes.c_double),
                ("abs_tol", ctypes.c_double), ("drop_tol", ctypes.c_double)]


class Diag(ctypes.Structure):
    _fields_ = [("solves", ctypes.c_int64 * 3), ("iterations", ctypes.c_int64 * 3),
                ("pcg_applies", ctypes.c_int64), ("maintenance_applies", ctypes.c_int64),
                ("basis_cols", ctypes.c_int32 * 3), ("pod_k", ctypes.c_int32),
                ("pod_info", ctypes.c_double), ("min_pod_info", ctypes.c_double),
                ("columns_accepted", ctypes.c_int64 * 3),
                ("columns_dropped", ctypes.c_int64 * 3),
                ("evictions", ctypes.c_int64 * 3)]


VP = ctypes.c_void_p
I32 = ctypes.c_int32
I64 = ctypes.c_int64
D = ctypes.c_double

# symbol -> (restype, argtypes); every entry point of include/mq_b200.h
SIGNATURES = {
    "mq_last_error": (ctypes.c_char_p, []),
    "mq_device_count": (I32, [c_int32_p]),
    "mq_device_sm_count": (I32, [I32, c_int32_p]),
    "mq_host_alloc": (I32, [I64, ctypes.POINTER(VP)]),
    "mq_host_free": (I32, [VP]),
    "mq_ctx_create": (I32, [ctypes.POINTER(GridDesc), I32, ctypes.POINTER(VP)]),
    "mq_ctx_destroy": (None, [VP]),
    "mq_n_n": (I64, [VP]),
    "mq_n_c": (I64, [VP]),
    "mq_dev_len": (I64, [VP]),
    "mq_kn_coefficients": (I32, [VP, c_double_p, c_double_p, c_double_p]),
    "mq_partition_export": (I32, [VP, c_int64_p, c_int64_p]),
    "mq_map_global_to_noncond": (I32, [VP, c_int64_p, I64, c_int64_p]),
    "mq_ctx_sync": (I32, [VP]),
    "mq_ctx_set_stream": (I32, [VP, VP]),
    "mq_ctx_set_sm_budget": (I32, [VP, I32]),
    "mq_pcg_kernel_info": (I32, [VP, ctypes.c_char_p, I32, c_int32_p]),
    "mq_vec_alloc": (I32, [VP, ctypes.POINTER(VP)]),
    "mq_vec_free": (I32, [VP, VP]),
    "mq_vec_upload": (I32, [VP, c_double_p, VP]),
    "mq_vec_download": (I32, [VP, VP, c_double_p]),
    "mq_kn_apply_dev": (I32, [VP, VP, VP]),
    "mq_kn_apply_host": (I32, [VP, c_double_p, c_double_p]),
    "mq_pcg_solve_dev": (I32, [VP, VP, VP, VP, D, D, I32, I32, ctypes.POINTER(SolveReportC)]),
    "mq_pcg_solve_host": (I32, [VP, c_double_p, c_double_p, c_double_p, D, D, I32, I32,
                                ctypes.POINTER(SolveReportC)]),
    "mq_csr_op_create": (I32, [I32, I64, I64, c_int64_p, c_int32_p, c_double_p, c_double_p, ctypes.POINTER(VP)]),
    "mq_csr_op_destroy": (I32, [VP]),
    "mq_csr_op_pcg": (I32, [VP, c_double_p, c_double_p, c_double_p, I32, D, D, I32,
                            ctypes.POINTER(SolveReportC)]),
    "mq_csr_op_spmv": (I32, [VP, c_double_p, c_double_p]),
    "mq_csr_pcg_solve": (I32, [I32, I64, c_int64_p, c_int32_p, c_double_p, c_double_p,
                               c_double_p, c_double_p, c_double_p, D, D, I32,
                               ctypes.POINTER(SolveReportC)]),
    "mq_csr_spmv": (I32, [I32, I64, I64, c_int64_p, c_int32_p, c_double_p, c_double_p,
                          c_double_p]),
    "mq_solver_init": (I32, [VP, ctypes.POINTER(SolverCfg), c_double_p]),
    "mq_solver_reset": (I32, [VP]),
    "mq_solve_kn": (I32, [VP, I32, VP, VP, ctypes.POINTER(SolveReportC)]),
    "mq_strategy_start": (I32, [VP, I32, VP, VP]),
    "mq_strategy_observe": (I32, [VP, I32, VP]),
    "mq_diagnostics": (I32, [VP, ctypes.POINTER(Diag)]),
    "mq_cspe_export": (I32, [VP, I32, c_int32_p, c_double_p, c_double_p, c_double_p]),
    "mq_kc_apply_host": (I32, [VP, c_double_p, c_double_p, c_double_p]),
    "mq_kcn_t_apply_host": (I32, [VP, c_double_p, c_double_p]),
    "mq_kcn_apply_host": (I32, [VP, c_double_p, c_double_p]),
    "mq_mc_diag": (I32, [VP, c_double_p]),
    "mq_state_set": (I32, [VP, c_double_p, D]),
    "mq_state_get": (I32, [VP, c_double_p, c_double_p]),
    "mq_euler_step": (I32, [VP, D, D, I64, ctypes.POINTER(SolveReportC),
                            ctypes.POINTER(SolveReportC)]),
    "mq_recover_an": (I32, [VP, D, c_double_p, ctypes.POINTER(SolveReportC),
                            ctypes.POINTER(SolveReportC)]),
    "mq_euler_step_host": (I32, [VP, c_double_p, D, D, D, I64, c_double_p, ctypes.POINTER(SolveReportC),
                                 ctypes.POINTER(SolveReportC)]),
    "mq_recover_an_host": (I32, [VP, c_double_p, D, D, c_double_p, ctypes.POINTER(SolveReportC),
                                 ctypes.POINTER(SolveReportC)]),
    "mq_last_an": (I32, [VP, c_double_p]),
    "mq_run_explicit": (I32, [VP, I64, c_double_p, c_double_p, I32, I32, c_int32_p,
                              c_double_p, c_int64_p]),
    "mq_run_explicit_states": (I32, [VP, I64, c_double_p, c_double_p, I32, I32, c_int32_p,
                                     c_double_p, c_double_p, c_int64_p]),
    "mq_run_prepare": (I32, [VP, I64, c_double_p, c_double_p, I32]),
    "mq_run_steps": (I32, [VP, I64, I32, VP]),
    "mq_run_finish": (I32, [VP, c_int32_p, c_int64_p]),
    "mq_probe_set": (I32, [VP, c_int64_p, I64]),
    "mq_probe_b": (I32, [VP, c_double_p, c_double_p]),
    "mq_run_probe_log": (I32, [VP, I64, c_double_p]),
    "mq_run_diag_log": (I32, [VP, I64, c_double_p]),
    "mq_pcg_collect": (I32, [VP, c_double_p, c_int32_p]),
    "mq_estimate_cfl": (I32, [VP, c_double_p, c_double_p, I32, D, D, D, I32, c_double_p,
                              c_double_p, c_int32_p, c_int64_p]),
    "mq_ctx_create_slab": (I32, [ctypes.POINTER(GridDesc), I32, I32, I32, ctypes.POINTER(VP)]),
    "mq_layout": (I32, [VP, c_int64_p]),
    "mq_slab_buffers": (I32, [VP, ctypes.POINTER(VP), ctypes.POINTER(VP), ctypes.POINTER(VP),
                              ctypes.POINTER(VP)]),
    "mq_slab_init": (I32, [VP, VP, VP, I32, I32, c_double_p]),
    "mq_slab_k1": (I32, [VP, VP, I32, D, D, I32, I32, c_double_p]),
    "mq_slab_k2": (I32, [VP, D, I32, c_double_p]),
    "mq_slab_final": (I32, [VP, VP, D, I32]),
    "mq_slab_ipc_export": (I32, [VP, VP, VP]),
    "mq_slab_ipc_import": (I32, [VP, I32, I32, VP, c_int32_p, VP]),
    "mq_slab_fused_solve_peer": (I32, [VP, VP, I32, D, D, I32, I32, ctypes.POINTER(SolveReportC)]),
    "mq_guard_check": (I32, [VP, c_int64_p, c_int32_p, c_int32_p]),
    "mq_pcg_solve_batched_host": (I32, [VP, I32, c_double_p, c_double_p, c_double_p, D, D, I32, I32,
                                       ctypes.POINTER(SolveReportC), c_double_p]),
    "mq_ss_init": (I32, [VP, ctypes.POINTER(SolverCfg), c_double_p]),
    "mq_ss_info": (I32, [VP, c_int64_p]),
    "mq_ss_owned": (I32, [VP, c_int64_p]),
    "mq_ss_vec": (I32, [VP, I32, ctypes.POINTER(VP)]),
    "mq_ss_state_set": (I32, [VP, c_double_p]),
    "mq_ss_state_get": (I32, [VP, c_double_p]),
    "mq_ss_rhs": (I32, [VP, I32, D]),
    "mq_ss_project": (I32, [VP, I32, I32, c_double_p]),
    "mq_ss_start": (I32, [VP, I32, c_double_p, VP]),
    "mq_ss_store": (I32, [VP, I32, VP, ctypes.POINTER(SolveReportC)]),
    "mq_ss_observe": (I32, [VP, I32, I32, c_double_p, c_double_p, c_int32_p]),
    "mq_ss_euler_prep": (I32, [VP]),
    "mq_ss_euler": (I32, [VP, D, c_double_p]),
    "mq_ss_an": (I32, [VP, c_double_p]),
    "mq_ss_diag": (I32, [VP, ctypes.POINTER(Diag)]),
    "mq_ss_cspe_export": (I32, [VP, I32, c_int32_p, c_double_p, c_double_p, c_double_p]),
    "mq_slab_fused_solve_local": (I32, [ctypes.POINTER(VP), I32, ctypes.POINTER(VP), ctypes.POINTER(VP), I32, D, D, I32, I32,
                                        ctypes.POINTER(SolveReportC)]),
    "mq_timer_start": (I32, [VP]),
    "mq_timer_stop": (I32, [VP, c_double_p]),
    "mq_pcg_stats": (I32, [VP, c_double_p, c_int64_p, c_int64_p, I32]),
    "mq_kernel_launches": (I32, [VP, c_int64_p]),
    "mq_pcg_trace": (I32, [VP, ctypes.POINTER(ctypes.c_uint64), I32]),
    "mq_l2_flush": (I32, [VP]),
}

_lib = None


def header_symbols() -> list[str]:
    """Entry points declared in include/mq_b200.h (parsed, for the tests)."""
    import re
    hdr = Path(__file__).resolve().parent.parent / "include" / "mq_b200.h"
    text = hdr.read_text()
    return sorted(set(re.findall(r"\b(mq_[a-z0-9_]+)\s*\(", text)))


def load(path: str | os.PathLike | None = None):
    """Load the shared library (once) and bind every signature."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else Path(os.environ.get("MQ_LIB_PATH", LIB_PATH))
    if not p.exists():
        raise RuntimeError(
            f"{p} is missing: the CUDA extension has not been built "
            "(run __graft_entry__.build()); there is no CPU fallback")
    lib = ctypes.CDLL(str(p))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib


class MqError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def last_error() -> str:
    return load().mq_last_error().decode("utf-8", "replace")


def check(rc: int, allow=(MQ_OK,)):
    """Map C return codes onto the reference's exception classes."""
    if rc in allow:
        return rc
    msg = last_error()
    if rc == MQ_INVALID:
        raise ValueError(msg)
    if rc == MQ_INDEFINITE:
        from .krylov import IndefiniteOperatorError
        raise IndefiniteOperatorError(msg)
    if rc in (MQ_NOT_CONVERGED, MQ_NONFINITE):
        from .schur import StepFailureError
        raise StepFailureError(msg)
    raise MqError(rc, f"libmq_b200 error {rc}: {msg}")


def dptr(a: np.ndarray):
    return a.ctypes.data_as(c_double_p)


def i64ptr(a: np.ndarray):
    return a.ctypes.data_as(c_int64_p)


def i32ptr(a: np.ndarray):
    return a.ctypes.data_as(c_int32_p)


def f64(a, n=None, name="vector") -> np.ndarray:
    v = np.ascontiguousarray(a, dtype=np.float64)
    if v.ndim != 1:
        raise ValueError(f"{name} must be one-dimensional, got shape {v.shape}")
    if n is not None and v.size != n:
        raise ValueError(f"{name} has length {v.size}, expected {n}")
    return v


def device_count() -> int:
    n = ctypes.c_int32(0)
    load().mq_device_count(ctypes.byref(n))
    return int(n.value)


def sm_count(device: int = 0) -> int:
    n = ctypes.c_int32(0)
    check(load().mq_device_sm_count(int(device), ctypes.byref(n)))
    return int(n.value)


class PinnedPool:
    """Page-locked float64 result arrays (mq_host_alloc), recycled by size.

    ``empty(n)`` returns a numpy array backed by pinned memory; when the
    array (and every view of it) is garbage collected, its buffer goes back
    to the pool instead of being freed, so steady-state calls allocate
    nothing and the device-to-host copy into it runs at DMA speed."""

    def __init__(self, max_free_per_size: int = 8):
        import threading
        self._free: dict[int, list[int]] = {}
        self._lock = threading.Lock()
        self._max = max_free_per_size

    def _release(self, n: int, ptr: int):
        with self._lock:
            lst = self._free.setdefault(n, [])
            if len(lst) < self._max:
                lst.append(ptr)
                return
        load().mq_host_free(ctypes.c_void_p(ptr))

    def reserve(self, n: int, count: int) -> None:
        """Have ``count`` free buffers of length n ready (page-locking costs
        milliseconds per buffer; a stepping loop should not pay it)."""
        with self._lock:
            have = len(self._free.get(n, []))
        for _ in range(max(0, min(count, self._max) - have)):
            p = ctypes.c_void_p()
            check(load().mq_host_alloc(8 * max(n, 1), ctypes.byref(p)))
            with self._lock:
                self._free.setdefault(n, []).append(p.value)

    def empty(self, n: int) -> np.ndarray:
        import weakref
        with self._lock:
            lst = self._free.get(n)
            ptr = lst.pop() if lst else None
        if ptr is None:
            p = ctypes.c_void_p()
            check(load().mq_host_alloc(8 * max(n, 1), ctypes.byref(p)))
            ptr = p.value
        buf = (ctypes.c_double * max(n, 1)).from_address(ptr)
        arr = np.frombuffer(buf, dtype=np.float64, count=n)
        weakref.finalize(arr, self._release, n, ptr)
        return arr


_PINNED = None


def _pool() -> PinnedPool:
    global _PINNED
    if _PINNED is None:
        _PINNED = PinnedPool()
    return _PINNED


def pinned_empty(n: int) -> np.ndarray:
    """float64 array of length n in recycled page-locked memory."""
    return _pool().empty(n)


def pinned_reserve(n: int, count: int = 4) -> None:
    """Pre-allocate ``count`` recycled page-locked buffers of length n."""
    _pool().reserve(n, count)
