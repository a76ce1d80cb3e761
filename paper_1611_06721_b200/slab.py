"""i-slab distributed K_n PCG (BASELINE configs[4]: 256^3 over 2/4/8 GPUs).

The node planes i = 0 .. nx-1 of the grid are split into contiguous slabs,
one per rank (the survey's "z-slabs": the slowest axis of the device layout,
which is the reference's i index).  Every rank owns the K_n dofs of its
planes; the stencil of a row at plane i touches planes i-1..i+1, so each
slab keeps one ghost plane per side.  Per PCG iteration (krylov.py:174-250):

    halo exchange of r and p_old ghost planes        (NCCL send/recv)
    K1 on the slab -> partial p.Ap                    allreduce(1)
    K2 on the slab -> partials r.r, r.z               allreduce(2)

The host loop below is shared by the GPU slabs (``SlabGrid``, phase kernels
in ``csrc/slab.cu``) and by any object with the same methods (the CPU tests
drive a numpy slab through it with gloo).  Communicators: ``TorchComm``
(torch.distributed; NCCL on GPUs, gloo on CPU) and ``LoopbackComm`` (several
slabs in one process: the single-GPU test of the decomposition).
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _lib
from ._lib import check, dptr, f64

__all__ = ["slab_range", "SlabGrid", "TorchComm", "LoopbackComm", "slab_pcg_solve", "fused_slab_pcg_solve_local",
           "gather_ipc_tables", "fused_peer_setup", "fused_peer_solve"]

IPC_HANDLE_BYTES = 9 * 64  # r, p_a, p_b, x, mailbox, counter, r2, ap, ap2 (cudaIpcMemHandle_t = 64 B)


def slab_range(nx: int, world: int, rank: int) -> tuple[int, int]:
    """Node planes [lo, hi) owned by ``rank`` (balanced contiguous split)."""
    if not (0 <= rank < world) or world > nx:
        raise ValueError("invalid slab decomposition")
    base, extra = divmod(nx, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


class _DevArray:
    """__cuda_array_interface__ view of device memory (for torch.as_tensor)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False),
                                         "version": 3, "strides": None}


class SlabGrid:
    """One i-slab of a Problem on a GPU (``mq_ctx_create_slab``)."""

    def __init__(self, problem, rank: int, world: int, device: int = 0):
        self.lib = _lib.load()
        mat = np.ascontiguousarray(problem.material, dtype=np.int8)
        self._mat = mat
        nx = mat.shape[0]
        self.rank, self.world = rank, world
        self.lo, self.hi = slab_range(nx, world, rank)
        k1, k2, k3 = problem.brauer
        desc = _lib.GridDesc(mat.shape[0], mat.shape[1], mat.shape[2], float(problem.h),
                             mat.ctypes.data_as(_lib.c_int8_p), float(problem.nu_air),
                             float(problem.kappa), float(k1), float(k2), float(k3),
                             float(problem.kn_diag), float(problem.kn_off))
        ctx = ctypes.c_void_p()
        check(self.lib.mq_ctx_create_slab(ctypes.byref(desc), self.lo, self.hi, int(device),
                                          ctypes.byref(ctx)))
        self.ctx = ctx
        self.device = device
        self.n_n = int(self.lib.mq_n_n(ctx))
        lay = np.zeros(6, dtype=np.int64)
        check(self.lib.mq_layout(ctx, _lib.i64ptr(lay)))
        self.C, self.Si, self.Sj, self.off, self.total, self.n_planes = (int(v) for v in lay)
        r, pa, pb, ap = (ctypes.c_void_p() for _ in range(4))
        check(self.lib.mq_slab_buffers(ctx, ctypes.byref(r), ctypes.byref(pa), ctypes.byref(pb),
                                       ctypes.byref(ap)))
        self.bufs = {"r": r.value, "pa": pa.value, "pb": pb.value}
        self.x = self.alloc()
        self.b = self.alloc()

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.mq_ctx_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def alloc(self) -> int:
        p = ctypes.c_void_p()
        check(self.lib.mq_vec_alloc(self.ctx, ctypes.byref(p)))
        return p.value

    def upload(self, host, dev: int):
        check(self.lib.mq_vec_upload(self.ctx, dptr(f64(host, self.n_n)), ctypes.c_void_p(dev)))

    def download(self, dev: int) -> np.ndarray:
        out = np.empty(self.n_n)
        check(self.lib.mq_vec_download(self.ctx, ctypes.c_void_p(dev), dptr(out)))
        return out

    def partition(self) -> np.ndarray:
        nc = np.empty(self.n_n, dtype=np.int64)
        check(self.lib.mq_partition_export(self.ctx, _lib.i64ptr(nc), None))
        return nc

    # -- halo planes: torch views of the device memory --------------------
    def _ptr(self, name):
        return self.x if name == "x" else self.bufs[name]

    def plane_views(self, name: str, plane: int):
        """torch CUDA views of local plane ``plane`` (-1 .. n) of vector ``name``,
        one per edge component."""
        import torch
        base = self._ptr(name)
        out = []
        for c in range(3):
            start = c * self.C + (plane + 1) * self.Si
            out.append(torch.as_tensor(_DevArray(base + 8 * start, self.Si), device=f"cuda:{self.device}"))
        return out

    def send_planes(self, name):
        return {"lo": self.plane_views(name, 0), "hi": self.plane_views(name, self.n_planes - 1)}

    def ghost_planes(self, name):
        return {"lo": self.plane_views(name, -1), "hi": self.plane_views(name, self.n_planes)}

    def sync(self):
        check(self.lib.mq_ctx_sync(self.ctx))

    def sync_torch(self):
        import torch
        torch.cuda.synchronize(self.device)

    # -- phases -------------------------------------------------------------
    def init(self, x0_mode: int, jac: bool) -> np.ndarray:
        part = np.zeros(3)
        check(self.lib.mq_slab_init(self.ctx, ctypes.c_void_p(self.b), ctypes.c_void_p(self.x),
                                    x0_mode, int(jac), dptr(part)))
        return part

    def k1(self, first, beta, alpha_prev, pold_is_a, jac) -> np.ndarray:
        part = np.zeros(1)
        check(self.lib.mq_slab_k1(self.ctx, ctypes.c_void_p(self.x), int(first), float(beta),
                                  float(alpha_prev), int(pold_is_a), int(jac), dptr(part)))
        return part

    def k2(self, alpha, jac) -> np.ndarray:
        part = np.zeros(2)
        check(self.lib.mq_slab_k2(self.ctx, float(alpha), int(jac), dptr(part)))
        return part

    def final(self, alpha, p_is_a):
        check(self.lib.mq_slab_final(self.ctx, ctypes.c_void_p(self.x), float(alpha), int(p_is_a)))


class LoopbackComm:
    """All slabs live in this process (in slab order): halos are device
    copies, allreduce is a fixed-order sum of the slabs' partials."""

    def allreduce(self, parts):
        tot = np.zeros_like(parts[0])
        for p in parts:
            tot = tot + p
        return [tot.copy() for _ in parts]

    def exchange(self, slabs, names):
        for name in names:
            for a, b in zip(slabs[:-1], slabs[1:]):
                # a's top owned plane -> b's low ghost; b's low owned plane -> a's top ghost
                for src, dst in zip(a.send_planes(name)["hi"], b.ghost_planes(name)["lo"]):
                    dst.copy_(src)
                for src, dst in zip(b.send_planes(name)["lo"], a.ghost_planes(name)["hi"]):
                    dst.copy_(src)
        for s in slabs:
            if hasattr(s, "sync_torch"):
                s.sync_torch()


class TorchComm:
    """One slab per rank; torch.distributed (NCCL for CUDA tensors, gloo for CPU)."""

    def __init__(self, dist, device=None):
        self.dist = dist
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()
        # gloo moves host memory only: device planes are staged through the host
        self.host_staged = dist.get_backend() == "gloo"
        self.device = "cpu" if self.host_staged else device

    def allreduce(self, parts):
        import torch
        (p,) = parts
        t = torch.tensor(p, dtype=torch.float64, device=self.device if self.device is not None else "cpu")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
        return [t.cpu().numpy()]

    def exchange(self, slabs, names):
        (s,) = slabs
        ops, land = [], []
        P2P = self.dist.P2POp

        def out(t):
            return t.cpu() if self.host_staged and t.is_cuda else t

        def into(t):
            if self.host_staged and t.is_cuda:
                h = t.new_empty(t.shape, device="cpu")
                land.append((t, h))
                return h
            return t

        for name in names:
            send, ghost = s.send_planes(name), s.ghost_planes(name)
            if self.rank > 0:
                for t in send["lo"]:
                    ops.append(P2P(self.dist.isend, out(t), self.rank - 1))
                for t in ghost["lo"]:
                    ops.append(P2P(self.dist.irecv, into(t), self.rank - 1))
            if self.rank + 1 < self.world:
                for t in send["hi"]:
                    ops.append(P2P(self.dist.isend, out(t), self.rank + 1))
                for t in ghost["hi"]:
                    ops.append(P2P(self.dist.irecv, into(t), self.rank + 1))
        if ops:
            for req in self.dist.batch_isend_irecv(ops):
                req.wait()
        for t, h in land:
            t.copy_(h)
        if hasattr(s, "sync_torch"):
            s.sync_torch()


def slab_pcg_solve(slabs, comm, *, x0_given: bool, rel_tol=1e-8, abs_tol=0.0, max_iter=5000,
                   jacobi=True):
    """krylov.py:174-250 over the slabs of this process.

    Right-hand side in each slab's ``b`` buffer, start vector (if
    ``x0_given``) in its ``x`` buffer; the solution is left in ``x``.
    Returns (iterations, final_rel_residual, converged, applications)."""
    if x0_given:
        comm.exchange(slabs, ["x"])
    parts = comm.allreduce([s.init(1 if x0_given else 2, jacobi) for s in slabs])
    bb, rr, rzs = (float(v) for v in parts[0])
    b_norm = math.sqrt(bb)
    target = max(rel_tol * b_norm, abs_tol)
    r_norm = math.sqrt(rr)
    applies = 1 if x0_given else 0

    def rel(v):
        if b_norm > 0.0:
            return v / b_norm
        return 0.0 if v == 0.0 else math.inf

    if r_norm <= target:
        return 0, rel(r_norm), True, applies
    rz = rzs if jacobi else rr
    beta = alpha_prev = alpha = 0.0
    first, pold_is_a = True, True
    for it in range(1, max_iter + 1):
        comm.exchange(slabs, ["r"] if first else ["r", "pa" if pold_is_a else "pb"])
        pap = float(comm.allreduce([s.k1(first, beta, alpha_prev, pold_is_a, jacobi) for s in slabs])[0][0])
        applies += 1
        if not math.isfinite(pap) or pap <= 0.0:
            from .krylov import IndefiniteOperatorError
            raise IndefiniteOperatorError(f"nonpositive curvature p^T A p = {pap:.3e} at iteration {it}")
        alpha = rz / pap
        rr, rz2 = (float(v) for v in comm.allreduce([s.k2(alpha, jacobi) for s in slabs])[0])
        r_norm = math.sqrt(rr)
        rz_new = rz2 if jacobi else rr
        p_new_is_a = not pold_is_a
        if r_norm <= target:
            for s in slabs:
                s.final(alpha, p_new_is_a)
            return it, rel(r_norm), True, applies
        if not math.isfinite(rz_new):
            from .krylov import IndefiniteOperatorError
            raise IndefiniteOperatorError(f"non-finite preconditioned residual at iteration {it}")
        beta = rz_new / rz
        rz = rz_new
        alpha_prev = alpha
        first = False
        pold_is_a = p_new_is_a
    for s in slabs:
        s.final(alpha, pold_is_a)
    return max_iter, rel(r_norm), False, applies


def fused_slab_pcg_solve_local(slabs, *, x0_given: bool, rel_tol=1e-8, abs_tol=0.0, max_iter=5000,
                               jacobi=True):
    """krylov.py:174-250 over the slabs of this process with the fused kernel
    (csrc/slab_fused.cu): ghost planes stored straight into the neighbour
    slab and the rank all-reduce through device mailboxes, one cooperative
    launch whose CTA groups are the ranks (the one-GPU form of the per-GPU
    kernel).  Right-hand sides in ``s.b``, start vectors in ``s.x``; the
    solution is left in ``s.x``.  Returns (iterations, final_rel_residual,
    converged, applications)."""
    from .krylov import IndefiniteOperatorError
    lib = slabs[0].lib
    n = len(slabs)
    ctxs = (ctypes.c_void_p * n)(*[s.ctx.value for s in slabs])
    bs = (ctypes.c_void_p * n)(*[s.b for s in slabs])
    xs = (ctypes.c_void_p * n)(*[s.x for s in slabs])
    rep = _lib.SolveReportC()
    rc = lib.mq_slab_fused_solve_local(ctxs, n, bs, xs, int(bool(x0_given)), float(rel_tol), float(abs_tol),
                                       int(max_iter), int(bool(jacobi)), ctypes.byref(rep))
    if rc == _lib.MQ_INDEFINITE:
        raise IndefiniteOperatorError(_lib.last_error())
    check(rc, allow=(0, 1))
    return int(rep.iterations), float(rep.final_rel_residual), bool(rep.converged), int(rep.applies)


def gather_ipc_tables(local_handles: bytes, local_planes: int, dist=None):
    """All-gather every rank's IPC handle block and owned plane count, in
    rank order (torch.distributed all_gather_object; identity for 1 rank)."""
    if len(local_handles) != IPC_HANDLE_BYTES:
        raise ValueError("unexpected IPC handle block size")
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return [local_handles], [int(local_planes)]
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, (local_handles, int(local_planes)))
    return [h for h, _ in out], [n for _, n in out]


def fused_peer_setup(slab: SlabGrid, dist=None):
    """Map the neighbour ranks' buffers (one rank per process and GPU) for
    :func:`fused_peer_solve` (mq_slab_ipc_export / import)."""
    rank = dist.get_rank() if dist is not None and dist.is_initialized() else 0
    world = dist.get_world_size() if dist is not None and dist.is_initialized() else 1
    buf = ctypes.create_string_buffer(IPC_HANDLE_BYTES)
    check(slab.lib.mq_slab_ipc_export(slab.ctx, ctypes.c_void_p(slab.x), buf))
    handles, planes = gather_ipc_tables(buf.raw, slab.n_planes, dist)
    allb = ctypes.create_string_buffer(b"".join(handles), IPC_HANDLE_BYTES * world)
    np_arr = (ctypes.c_int32 * world)(*planes)
    check(slab.lib.mq_slab_ipc_import(slab.ctx, rank, world, allb, np_arr, ctypes.c_void_p(slab.x)))


def fused_peer_solve(slab: SlabGrid, *, x0_given: bool, rel_tol=1e-8, abs_tol=0.0, max_iter=5000, jacobi=True):
    """This rank's part of the fused distributed solve (every rank calls it):
    right-hand side in ``slab.b``, start vector / solution in ``slab.x``.
    Returns (iterations, final_rel_residual, converged, applications)."""
    from .krylov import IndefiniteOperatorError
    rep = _lib.SolveReportC()
    rc = slab.lib.mq_slab_fused_solve_peer(slab.ctx, ctypes.c_void_p(slab.b), int(bool(x0_given)), float(rel_tol),
                                           float(abs_tol), int(max_iter), int(bool(jacobi)), ctypes.byref(rep))
    if rc == _lib.MQ_INDEFINITE:
        raise IndefiniteOperatorError(_lib.last_error())
    check(rc, allow=(0, 1))
    return int(rep.iterations), float(rep.final_rel_residual), bool(rep.converged), int(rep.applies)
