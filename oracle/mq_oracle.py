"""CPU oracle for the mq-b200 hot path — TEST INFRASTRUCTURE ONLY.

This module is the parity checker. Only ``tests/``, ``__graft_entry__.smoke()``
and the ``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import
it. The product (``paper_1611_06721_b200``) never routes through it.

It restates, in plain numpy/scipy, the reference algorithm of the path that
BASELINE.json's north star names (reference = ``mqsolve``, paths relative to
``/root/reference/pkg/src/mqsolve``):

* FIT edge topology, PEC boundary, conducting-edge rule, partition
  (``model.py:186-272``, ``model.py:438-470``)
* ``K_n``, ``K_cn``, ``M_c`` assembly (``model.py:472-491``)
* Brauer ``K_c(a) x`` (``model.py:107-125``, ``model.py:492-509``)
* closed-loop coil source patterns (``model.py:321-336``, ``model.py:529-556``)
* PCG with Jacobi (``krylov.py:82-97``, ``krylov.py:174-250``)
* SPE/CSPE subspace cache (``startvec.py:59-79``, ``startvec.py:118-225``)
* POD snapshots (``startvec.py:239-309``) and the three strategies
  (``startvec.py:345-472``)
* ``solve_kn`` / explicit Euler / recovery / time loop (``schur.py:239-264``,
  ``schur.py:379-419``, ``schur.py:474-607``) and the CFL power iteration
  (``schur.py:327-376``).

The numerics deliberately follow the reference's numpy/scipy call sequence so
that, on the same inputs, the oracle reproduces the reference bit for bit.
That is pinned by ``tests/test_oracle_golden.py`` against fixtures produced by
running the reference itself (``tests/golden/make_golden.py``).

The numpy/scipy arithmetic boundary (scipy ``sparsetools`` SpMV, OpenBLAS
dot/gemv, LAPACK ``syevd``/``trtrs``) is not vendored by the reference and is
unpinned there (``pkg/pyproject.toml:10-13`` lists ``numpy>=1.24``,
``scipy>=1.10``); the goldens were produced with numpy 2.3.5 / scipy 1.18.1.
"""

from __future__ import annotations

import math
from collections import deque
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg
import scipy.sparse as sp

NU_VACUUM = 1.0 / (4e-7 * np.pi)          # model.py:63
AIR, CONDUCTOR, COIL = 0, 1, 2            # model.py:61

FAM_SOURCE = "source"                     # startvec.py:45-50
FAM_CUR = "coupling_current"
FAM_PREV = "coupling_previous"
FAMILY_ORDER = (FAM_SOURCE, FAM_CUR, FAM_PREV)


class OracleIndefinite(RuntimeError):
    """krylov.py:44-45 (IndefiniteOperatorError)."""


class OracleStepFailure(RuntimeError):
    """schur.py:56-57 (StepFailureError)."""


# ---------------------------------------------------------------------------
# edge / face numbering  (model.py:186-207)
# ---------------------------------------------------------------------------


class Numbering:
    """Global edge, face and cell ids of an nx*ny*nz cell grid, k fastest."""

    def __init__(self, nx: int, ny: int, nz: int):
        self.shape = (nx, ny, nz)
        sx = (nx, ny + 1, nz + 1)
        sy = (nx + 1, ny, nz + 1)
        sz = (nx + 1, ny + 1, nz)
        self.edge_shapes = (sx, sy, sz)
        cnt = [int(np.prod(s)) for s in self.edge_shapes]
        self.edge_offsets = (0, cnt[0], cnt[0] + cnt[1])
        self.n_edges = sum(cnt)
        self.edge_ids = tuple(
            off + np.arange(c).reshape(s)
            for off, c, s in zip(self.edge_offsets, cnt, self.edge_shapes))
        fs = ((nx + 1, ny, nz), (nx, ny + 1, nz), (nx, ny, nz + 1))
        fc = [int(np.prod(s)) for s in fs]
        foff = (0, fc[0], fc[0] + fc[1])
        self.n_faces = sum(fc)
        self.face_ids = tuple(
            off + np.arange(c).reshape(s) for off, c, s in zip(foff, fc, fs))
        self.n_cells = nx * ny * nz
        self.n_nodes = (nx + 1) * (ny + 1) * (nz + 1)
        self.node_ids = np.arange(self.n_nodes).reshape(nx + 1, ny + 1, nz + 1)

    # face -> its four edges with circulation signs (+,+,-,-), model.py:209-238
    def curl(self) -> sp.csr_matrix:
        nx, ny, nz = self.shape
        ex, ey, ez = self.edge_ids
        fx, fy, fz = self.face_ids
        quads = (
            (fx, (ey[:, :, :nz], ez[:, 1:, :], ey[:, :, 1:], ez[:, :ny, :])),
            (fy, (ez[:nx, :, :], ex[:, :, 1:], ez[1:, :, :], ex[:, :, :nz])),
            (fz, (ex[:, :ny, :], ey[1:, :, :], ex[:, 1:, :], ey[:nx, :, :])),
        )
        r, c, v = [], [], []
        for faces, edges in quads:
            nf = faces.size
            r.append(np.repeat(faces.reshape(-1), 4))
            c.append(np.stack([e.reshape(-1) for e in edges], axis=1).reshape(-1))
            v.append(np.tile(np.array([1.0, 1.0, -1.0, -1.0]), nf))
        m = sp.coo_matrix((np.concatenate(v), (np.concatenate(r), np.concatenate(c))),
                          shape=(self.n_faces, self.n_edges)).tocsr()
        m.sort_indices()
        return m

    # PEC: edges lying in a boundary plane, model.py:240-251
    def on_boundary(self) -> np.ndarray:
        nx, ny, nz = self.shape
        out = []
        for comp, shp in enumerate(self.edge_shapes):
            flag = np.zeros(shp, dtype=bool)
            for ax in range(3):
                if ax == comp:
                    continue
                last = (nx, ny, nz)[ax]
                idx = [slice(None)] * 3
                idx[ax] = [0, last]
                flag[tuple(idx)] = True
            out.append(flag.reshape(-1))
        return np.concatenate(out)

    def _four_cells(self, cells: np.ndarray, comp: int):
        """The four (zero-padded) cells around every edge of one component."""
        pad = [(1, 1)] * 3
        pad[comp] = (0, 0)
        p = np.pad(cells, pad)
        a, b = [d for d in range(3) if d != comp]
        views = []
        for da in (0, 1):
            for db in (0, 1):
                sl = [slice(None)] * 3
                sl[a] = slice(da, p.shape[a] - 1 + da)
                sl[b] = slice(db, p.shape[b] - 1 + db)
                views.append(p[tuple(sl)])
        return views

    # conducting rule: edge borders >= 1 conductor cell, model.py:253-272
    def touches(self, cell_mask: np.ndarray) -> np.ndarray:
        out = []
        for comp in range(3):
            v = self._four_cells(cell_mask, comp)
            out.append((v[0] | v[1] | v[2] | v[3]).reshape(-1))
        return np.concatenate(out)

    # mean of the four adjacent cell values, model.py:274-292
    def edge_mean(self, cell_values: np.ndarray) -> np.ndarray:
        out = []
        for comp in range(3):
            v = self._four_cells(cell_values.astype(np.float64), comp)
            out.append(((((v[0] + v[1]) + v[2]) + v[3]) / 4.0).reshape(-1))
        return np.concatenate(out)

    # 0.5 per adjacent cell, cells -> faces, model.py:294-310
    def face_average(self) -> sp.csr_matrix:
        nx, ny, nz = self.shape
        cid = np.arange(self.n_cells).reshape(nx, ny, nz)
        fx, fy, fz = self.face_ids
        r = [fx[1:], fx[:nx], fy[:, 1:], fy[:, :ny], fz[:, :, 1:], fz[:, :, :nz]]
        r = np.concatenate([x.reshape(-1) for x in r])
        c = np.concatenate([cid.reshape(-1)] * 6)
        return sp.coo_matrix((np.full(r.size, 0.5), (r, c)),
                             shape=(self.n_faces, self.n_cells)).tocsr()

    # per cell: x pair, y pair, z pair of faces, model.py:312-319
    def cell_faces(self) -> np.ndarray:
        nx, ny, nz = self.shape
        fx, fy, fz = self.face_ids
        six = np.stack([fx[:nx], fx[1:], fy[:, :ny], fy[:, 1:],
                        fz[:, :, :nz], fz[:, :, 1:]], axis=-1)
        return six.reshape(self.n_cells, 6)

    # rectangular loop in a z node plane, model.py:321-336
    def loop(self, i0, i1, j0, j1, k0):
        ex, ey, _ = self.edge_ids
        ids = np.concatenate([ex[i0:i1, j0, k0], ey[i1, j0:j1, k0],
                              ex[i0:i1, j1, k0], ey[i0, j0:j1, k0]])
        sg = np.concatenate([np.ones(i1 - i0), np.ones(j1 - j0),
                             -np.ones(i1 - i0), -np.ones(j1 - j0)])
        return ids, sg

    def edge_tail_head(self):
        nx, ny, nz = self.shape
        n = self.node_ids
        tails = np.concatenate([n[:nx].reshape(-1), n[:, :ny].reshape(-1),
                                n[:, :, :nz].reshape(-1)])
        heads = np.concatenate([n[1:].reshape(-1), n[:, 1:].reshape(-1),
                                n[:, :, 1:].reshape(-1)])
        return tails, heads


# ---------------------------------------------------------------------------
# assembly (model.py:438-579), generalised to a list of closed loops
# ---------------------------------------------------------------------------


@dataclass
class Conductor:
    kappa: float
    k1: float = 0.0
    k2: float = 0.0
    k3: float = NU_VACUUM

    @property
    def linear(self) -> bool:
        return self.k1 == 0.0


def brauer_nu(cond: Conductor, b2: np.ndarray) -> np.ndarray:
    """model.py:107-125: nu = k1 exp(k2 B^2) + k3 (overflow ignored)."""
    if cond.linear:
        return np.full_like(b2, cond.k3)
    with np.errstate(over="ignore"):
        return cond.k1 * np.exp(cond.k2 * b2) + cond.k3


@dataclass
class Loop:
    i0: int
    i1: int
    j0: int
    j1: int
    k0: int
    amps: float


@dataclass
class OracleModel:
    shape: tuple
    h: float
    nu_air: float
    conductor: Conductor
    material: np.ndarray
    interior: np.ndarray          # global ids of retained edges
    cond: np.ndarray              # positions (interior order) of conducting dofs
    noncond: np.ndarray
    kn: sp.csr_matrix
    kcn: sp.csr_matrix
    mc_diag: np.ndarray
    pattern: np.ndarray
    kc_apply: object
    c_int: sp.csr_matrix
    cell_faces: np.ndarray
    cond_cells: np.ndarray

    @property
    def n_c(self):
        return int(self.cond.size)

    @property
    def n_n(self):
        return int(self.noncond.size)

    @property
    def noncond_global(self):
        return self.interior[self.noncond]

    @property
    def cond_global(self):
        return self.interior[self.cond]

    def kn_apply(self, x):
        return self.kn @ x


def assemble(material: np.ndarray, h: float, conductor: Conductor,
             loops: list[Loop], nu_air: float = NU_VACUUM) -> OracleModel:
    """Partitioned FIT system; the connectivity check of model.py:428-435 is
    not applied (configs 2 and 4 carry two disjoint iron blocks)."""
    nx, ny, nz = material.shape
    num = Numbering(nx, ny, nz)
    cmask = material == CONDUCTOR
    if not cmask.any():
        raise ValueError("no conductor cells")
    interior = np.flatnonzero(~num.on_boundary())
    pos = np.full(num.n_edges, -1, dtype=np.int64)
    pos[interior] = np.arange(interior.size)
    cond_glob = num.touches(cmask)
    cond = np.flatnonzero(cond_glob[interior])
    noncond = np.flatnonzero(~cond_glob[interior])

    c_int = num.curl()[:, interior].tocsr()
    c_cond = c_int[:, cond].tocsr()
    avg = num.face_average()
    six = num.cell_faces()
    ccells = np.flatnonzero(cmask.reshape(-1))
    avg_c = avg[:, ccells].tocsr()
    base = avg @ np.where(cmask.reshape(-1), 0.0, nu_air)
    w0 = base + avg_c @ np.full(ccells.size, conductor.k1 + conductor.k3)
    k_all = (c_int.T @ sp.diags(w0 / h) @ c_int).tocsr()
    kcn = _canonical(k_all[cond][:, noncond])
    kn = _canonical(k_all[noncond][:, noncond])

    kap = num.edge_mean(np.where(cmask, conductor.kappa, 0.0))
    mc_diag = kap[interior][cond] * h
    if (mc_diag <= 0).any():
        raise ValueError("conducting edge without conductivity")

    faces_c = six[ccells]
    two_h4 = 2.0 * (h ** 4)

    def kc_apply(state, x):
        phi = c_cond @ np.asarray(state, dtype=np.float64)
        f = phi[faces_c]
        b2 = ((f[:, 0] ** 2 + f[:, 1] ** 2) + (f[:, 2] ** 2 + f[:, 3] ** 2)
              + (f[:, 4] ** 2 + f[:, 5] ** 2)) / two_h4
        w = base + avg_c @ brauer_nu(conductor, b2)
        return c_cond.T @ ((w / h) * (c_cond @ np.asarray(x, dtype=np.float64)))

    # source: sum of closed loops, each checked like model.py:529-556
    tails, heads = num.edge_tail_head()
    nidx = np.full(interior.size, -1, dtype=np.int64)
    nidx[noncond] = np.arange(noncond.size)
    pattern = np.zeros(noncond.size)
    for lp in loops:
        ids, sg = num.loop(lp.i0, lp.i1, lp.j0, lp.j1, lp.k0)
        div = np.zeros(num.n_nodes)
        np.add.at(div, heads[ids], sg)
        np.add.at(div, tails[ids], -sg)
        if np.abs(div).max() > 0:
            raise ValueError("loop not closed")
        p = pos[ids]
        if (p < 0).any() or cond_glob[ids].any():
            raise ValueError("loop touches boundary or conducting edges")
        one = np.zeros(noncond.size)
        np.add.at(one, nidx[p], sg * lp.amps)
        pattern = pattern + one
    return OracleModel(shape=(nx, ny, nz), h=h, nu_air=nu_air,
                       conductor=conductor, material=material,
                       interior=interior, cond=cond, noncond=noncond, kn=kn,
                       kcn=kcn, mc_diag=mc_diag, pattern=pattern,
                       kc_apply=kc_apply, c_int=c_int, cell_faces=six,
                       cond_cells=ccells)


def _canonical(m) -> sp.csr_matrix:
    """sparse.py:123-128 (CsrMatrix.from_scipy canonical form)."""
    c = sp.csr_matrix(m)
    c.sum_duplicates()
    c.sort_indices()
    return c


def cell_b2(model: OracleModel, a_interior) -> np.ndarray:
    """model.py:399-407: squared cell flux density."""
    phi = model.c_int @ np.asarray(a_interior, dtype=np.float64)
    f = phi[model.cell_faces]
    return ((f[:, 0] ** 2 + f[:, 1] ** 2) + (f[:, 2] ** 2 + f[:, 3] ** 2)
            + (f[:, 4] ** 2 + f[:, 5] ** 2)) / (2.0 * model.h ** 4)


def full_interior(model: OracleModel, a_c, a_n) -> np.ndarray:
    """model.py:385-391: scatter (a_c, a_n) into the interior vector."""
    full = np.zeros(model.interior.size)
    full[model.cond] = a_c
    full[model.noncond] = a_n
    return full


def default_probe_cells(model: OracleModel, shape) -> np.ndarray:
    """model.py:562-566: conductor cells in the median k layer (global ids)."""
    nx, ny, nz = shape
    ijk = np.stack(np.unravel_index(model.cond_cells, (nx, ny, nz)), axis=1)
    mid_k = int(np.median(ijk[:, 2]))
    sel = ijk[ijk[:, 2] == mid_k]
    return (sel[:, 0] * ny + sel[:, 1]) * nz + sel[:, 2]


def probe_b(model: OracleModel, a_interior, cells) -> float:
    """model.py:415-425: mean |B| over the probe cells."""
    b2 = cell_b2(model, a_interior)
    return float(np.sqrt(b2[np.asarray(cells, dtype=np.int64)]).mean())


# ---------------------------------------------------------------------------
# PCG  (krylov.py:82-97, 174-250)
# ---------------------------------------------------------------------------


@dataclass
class PcgResult:
    x: np.ndarray
    iterations: int
    rel: float
    converged: bool
    applies: int


def jacobi_inverse(diag: np.ndarray) -> np.ndarray:
    d = np.asarray(diag, dtype=np.float64)
    return np.where(d > 0, 1.0 / np.where(d > 0, d, 1.0), 1.0)


def pcg(apply_a, b, x0=None, rel_tol=1e-8, abs_tol=0.0, max_iter=5000,
        inv_diag=None) -> PcgResult:
    b = np.asarray(b, dtype=np.float64)
    nb = float(np.linalg.norm(b))
    target = max(rel_tol * nb, abs_tol)
    n_app = 0
    if x0 is None:
        x = np.zeros_like(b)
        r = b.copy()
    else:
        x = np.asarray(x0, dtype=np.float64).copy()
        r = b - apply_a(x)
        n_app += 1
    rn = float(np.linalg.norm(r))

    def rel(v):
        if nb > 0.0:
            return v / nb
        return 0.0 if v == 0.0 else np.inf

    if rn <= target:
        return PcgResult(x, 0, rel(rn), True, n_app)
    z = inv_diag * r if inv_diag is not None else r
    p = z.copy()
    rz = float(r @ z)
    for it in range(1, max_iter + 1):
        ap = apply_a(p)
        n_app += 1
        pap = float(p @ ap)
        if not np.isfinite(pap) or pap <= 0.0:
            raise OracleIndefinite(f"p^T A p = {pap!r} at iteration {it}")
        alpha = rz / pap
        x = x + alpha * p
        r = r - alpha * ap
        rn = float(np.linalg.norm(r))
        if rn <= target:
            return PcgResult(x, it, rel(rn), True, n_app)
        z = inv_diag * r if inv_diag is not None else r
        rz_new = float(r @ z)
        if not np.isfinite(rz_new):
            raise OracleIndefinite(f"non-finite r^T z at iteration {it}")
        p = z + (rz_new / rz) * p
        rz = rz_new
    return PcgResult(x, max_iter, rel(rn), False, n_app)


# ---------------------------------------------------------------------------
# small dense SPD helpers  (startvec.py:53-79)
# ---------------------------------------------------------------------------


class PivotFail(Exception):
    def __init__(self, j):
        super().__init__(j)
        self.j = j


def chol_lower(g: np.ndarray, floor: float = 1e-12) -> np.ndarray:
    n = g.shape[0]
    lo = np.zeros_like(g)
    for j in range(n):
        s = g[j, j] - lo[j, :j] @ lo[j, :j]
        if not np.isfinite(s) or s <= floor * abs(g[j, j]) or s <= 0.0:
            raise PivotFail(j)
        lo[j, j] = np.sqrt(s)
        if j + 1 < n:
            lo[j + 1:, j] = (g[j + 1:, j] - lo[j + 1:, :j] @ lo[j, :j]) / lo[j, j]
    return lo


def chol_solve(lo: np.ndarray, rhs: np.ndarray) -> np.ndarray:
    y = scipy.linalg.solve_triangular(lo, rhs, lower=True)
    return scipy.linalg.solve_triangular(lo.T, y, lower=False)


# ---------------------------------------------------------------------------
# SPE / CSPE cache  (startvec.py:118-225)
# ---------------------------------------------------------------------------


class SpeCache:
    def __init__(self, n, apply_a, max_cols=20, drop_tol=1e-10):
        self.n, self.apply_a = n, apply_a
        self.max_cols, self.drop_tol = max_cols, drop_tol
        self.U = np.empty((n, 0))
        self.KU = np.empty((n, 0))
        self.G = np.empty((0, 0))
        self.products = 0
        self.accepted = 0
        self.dropped = 0
        self.evictions = 0

    @property
    def k(self):
        return self.U.shape[1]

    def insert(self, v) -> bool:
        v = np.asarray(v, dtype=np.float64)
        nv = np.linalg.norm(v)
        if nv == 0.0 or not np.isfinite(nv):
            self.dropped += 1
            return False
        w = v.copy()
        for _ in range(2):
            if self.k:
                w -= self.U @ (self.U.T @ w)
        nw = np.linalg.norm(w)
        if nw < self.drop_tol * nv:
            self.dropped += 1
            return False
        u = w / nw
        if self.k == self.max_cols:
            self.U, self.KU, self.G = self.U[:, 1:], self.KU[:, 1:], self.G[1:, 1:]
            self.evictions += 1
        ku = np.asarray(self.apply_a(u), dtype=np.float64)
        self.products += 1
        cross = self.U.T @ ku
        k = self.k
        g = np.empty((k + 1, k + 1))
        g[:k, :k] = self.G
        g[:k, k] = cross
        g[k, :k] = cross
        g[k, k] = float(u @ ku)
        self.U = np.column_stack([self.U, u])
        self.KU = np.column_stack([self.KU, ku])
        self.G = g
        self.accepted += 1
        return True

    def _drop(self, j):
        keep = [i for i in range(self.k) if i != j]
        self.U, self.KU = self.U[:, keep], self.KU[:, keep]
        self.G = self.G[np.ix_(keep, keep)]

    def project(self, rhs) -> np.ndarray:
        rhs = np.asarray(rhs, dtype=np.float64)
        while self.k:
            beta = self.U.T @ rhs
            try:
                lo = chol_lower(self.G)
            except PivotFail as bad:
                self._drop(bad.j)
                self.dropped += 1
                continue
            return self.U @ chol_solve(lo, beta)
        return np.zeros(self.n)


# ---------------------------------------------------------------------------
# POD  (startvec.py:239-309)
# ---------------------------------------------------------------------------


class Snapshots:
    def __init__(self, n, n_pod=10, eps_pod=1e-4):
        self.n, self.eps = n, eps_pod
        self.ring = deque(maxlen=n_pod)

    def push(self, v):
        self.ring.append(np.asarray(v, dtype=np.float64).copy())

    def matrix(self):
        if not self.ring:
            return np.empty((self.n, 0))
        return np.column_stack(list(self.ring))


def pod_start(snap: Snapshots, rhs, apply_a):
    """Returns (x0, k, info, applications)."""
    rhs = np.asarray(rhs, dtype=np.float64)
    X = snap.matrix()
    if X.shape[1] == 0:
        return np.zeros(snap.n), 0, 0.0, 0
    lam, vec = np.linalg.eigh(X.T @ X)
    order = np.argsort(lam)[::-1]
    sig = np.sqrt(np.clip(lam[order], 0.0, None))
    vec = vec[:, order]
    if sig[0] == 0.0:
        return np.zeros(snap.n), 0, 0.0, 0
    k = int(np.count_nonzero(sig / sig[0] > snap.eps))
    total = float(sig.sum())
    B = (X @ vec[:, :k]) / sig[:k]
    KB = np.column_stack([np.asarray(apply_a(B[:, j]), dtype=np.float64)
                          for j in range(k)])
    applications = k
    while k:
        g = B[:, :k].T @ KB[:, :k]
        g = 0.5 * (g + g.T)
        try:
            lo = chol_lower(g)
        except PivotFail:
            k -= 1
            continue
        coef = chol_solve(lo, B[:, :k].T @ rhs)
        return B[:, :k] @ coef, k, float(sig[:k].sum() / total), applications
    return np.zeros(snap.n), 0, 0.0, applications


# ---------------------------------------------------------------------------
# strategies  (startvec.py:315-472)
# ---------------------------------------------------------------------------


class Strategy:
    kind = "zero"

    def __init__(self, n):
        self.n = n

    def start(self, fam, rhs):
        return np.zeros(self.n)

    def observe(self, fam, y):
        pass

    def basis_size(self):
        return 0

    @property
    def maintenance(self):
        return 0

    def diagnostics(self):
        return {}


class PreviousStrategy(Strategy):
    kind = "previous"

    def __init__(self, n):
        super().__init__(n)
        self.last = {}

    def start(self, fam, rhs):
        v = self.last.get(fam)
        return np.zeros(self.n) if v is None else v.copy()

    def observe(self, fam, y):
        self.last[fam] = np.asarray(y, dtype=np.float64).copy()


class CspeStrategyOracle(Strategy):
    kind = "cspe"

    def __init__(self, n, apply_a, max_cols=20, drop_tol=1e-10):
        super().__init__(n)
        self.apply_a, self.max_cols, self.drop_tol = apply_a, max_cols, drop_tol
        self.caches = {}

    def cache(self, fam):
        if fam not in self.caches:
            self.caches[fam] = SpeCache(self.n, self.apply_a, self.max_cols,
                                        self.drop_tol)
        return self.caches[fam]

    def start(self, fam, rhs):
        return self.cache(fam).project(rhs)

    def observe(self, fam, y):
        self.cache(fam).insert(y)

    def basis_size(self):
        return max((c.k for c in self.caches.values()), default=0)

    @property
    def maintenance(self):
        return sum(c.products for c in self.caches.values())

    def diagnostics(self):
        return {"basis_cols": self.basis_size(),
                "maintenance_applies": self.maintenance}


class PodStrategyOracle(Strategy):
    kind = "pod"

    def __init__(self, n, apply_a, n_pod=10, eps_pod=1e-4):
        super().__init__(n)
        self.apply_a, self.n_pod, self.eps_pod = apply_a, n_pod, eps_pod
        self.bufs = {}
        self.applies = 0
        self.last_k, self.last_info, self.min_info = 0, 1.0, 1.0
        self.any = False

    def buf(self, fam):
        if fam not in self.bufs:
            self.bufs[fam] = Snapshots(self.n, self.n_pod, self.eps_pod)
        return self.bufs[fam]

    def start(self, fam, rhs):
        b = self.buf(fam)
        if not b.ring:
            return np.zeros(self.n)
        x0, k, info, app = pod_start(b, rhs, self.apply_a)
        self.applies += app
        self.last_k, self.last_info = k, info
        if k:
            self.any = True
            self.min_info = min(self.min_info, info)
        return x0

    def observe(self, fam, y):
        self.buf(fam).push(y)

    def basis_size(self):
        return self.last_k

    @property
    def maintenance(self):
        return self.applies

    def diagnostics(self):
        return {"pod_k": self.last_k, "pod_info": self.last_info,
                "min_pod_info": self.min_info if self.any else 1.0,
                "maintenance_applies": self.applies}


def make_strategy(kind, n, apply_a, *, max_cols=20, n_pod=10, eps_pod=1e-4,
                  drop_tol=1e-10) -> Strategy:
    kind = kind.lower()
    if kind == "previous":
        return PreviousStrategy(n)
    if kind == "zero":
        return Strategy(n)
    if kind == "cspe":
        return CspeStrategyOracle(n, apply_a, max_cols, drop_tol)
    if kind == "pod":
        return PodStrategyOracle(n, apply_a, n_pod, eps_pod)
    raise ValueError(kind)


# ---------------------------------------------------------------------------
# Schur stepping  (schur.py:239-264, 266-287, 327-419, 474-607)
# ---------------------------------------------------------------------------


@dataclass
class CsrModel:
    """PartitionedSystem.linear (schur.py:85-160) of CSR blocks, as
    bench.py:228-313 loads a manifest without builtin parameters: the fields
    SchurOracle reads.  K_c is the stored (frozen) matrix."""
    kn: sp.csr_matrix
    kcn: sp.csr_matrix
    kc: sp.csr_matrix
    mc_diag: np.ndarray
    pattern: np.ndarray

    @property
    def n_c(self):
        return int(self.kcn.shape[0])

    @property
    def n_n(self):
        return int(self.kcn.shape[1])

    def kn_apply(self, x):
        return self.kn @ x

    def kc_apply(self, state, x):
        return self.kc @ x


class SchurOracle:
    """Owns the strategy and bookkeeping of every K_n solve."""

    def __init__(self, model: OracleModel, waveform, strategy="cspe",
                 rel_tol=1e-8, max_iter=5000, max_cols=20, n_pod=10,
                 eps_pod=1e-4):
        self.m = model
        self.waveform = waveform
        self.rel_tol, self.max_iter = rel_tol, max_iter
        self.inv = jacobi_inverse(model.kn.diagonal())
        self.strategy = make_strategy(strategy, model.n_n, model.kn_apply,
                                      max_cols=max_cols, n_pod=n_pod,
                                      eps_pod=eps_pod, drop_tol=rel_tol)
        self.minv_diag = 1.0 / model.mc_diag
        self.iters = {f: [] for f in FAMILY_ORDER}
        self.pcg_applies = 0

    def solve(self, rhs, fam):
        x0 = self.strategy.start(fam, rhs)
        res = pcg(self.m.kn_apply, rhs, x0=x0, rel_tol=self.rel_tol,
                  max_iter=self.max_iter, inv_diag=self.inv)
        if not res.converged:
            raise OracleStepFailure(f"{fam} stalled at {res.rel:.3e}")
        self.pcg_applies += res.applies
        self.strategy.observe(fam, res.x)
        self.iters[fam].append(res.iterations)
        return res.x, res

    def source_solve(self, t):
        return self.solve(self.m.pattern * float(self.waveform(t)), FAM_SOURCE)

    def euler(self, a_c, t, dt, step_index=None):
        if dt < 0:
            raise ValueError("dt must be nonnegative")
        t_new = t + dt
        y_src, r1 = self.source_solve(t_new)
        y_cpl, r2 = self.solve(self.m.kcn.T @ a_c, FAM_PREV)
        rate = self.m.kcn @ (y_cpl - y_src) - self.m.kc_apply(a_c, a_c)
        a_next = a_c + dt * (self.minv_diag * rate)
        if not np.isfinite(a_next).all():
            raise OracleStepFailure(f"non-finite state at step {step_index}")
        return a_next, (r1, r2)

    def recover(self, a_c, t):
        y_src, r1 = self.source_solve(t)
        y_cpl, r2 = self.solve(self.m.kcn.T @ a_c, FAM_CUR)
        return y_src - y_cpl, (r1, r2)

    # schur.py:297-313 + 327-376 (a_c_ref defaults to zero)
    def estimate_cfl(self, power_iters=200, power_tol=1e-4, safety=0.9,
                     seed=42, a_ref=None):
        n = self.m.n_c
        ref = np.zeros(n) if a_ref is None else a_ref
        v = np.random.default_rng(seed).standard_normal(n)
        v /= np.linalg.norm(v)
        lam, lam_prev, inner, used = 0.0, None, None, power_iters
        for it in range(1, power_iters + 1):
            w_n = self.m.kcn.T @ v
            res = pcg(self.m.kn_apply, w_n, x0=inner, rel_tol=self.rel_tol,
                      max_iter=self.max_iter, inv_diag=self.inv)
            if not res.converged:
                raise OracleStepFailure("spectral probe stalled")
            self.pcg_applies += res.applies
            inner = res.x
            w = self.m.kc_apply(ref, v) - self.m.kcn @ inner
            lam = float(v @ w) / float(v @ (self.m.mc_diag * v))
            u = self.minv_diag * w
            nu = np.linalg.norm(u)
            v = u / nu
            if lam_prev is not None and abs(lam - lam_prev) <= power_tol * abs(lam):
                used = it
                break
            lam_prev = lam
        return lam, safety * 2.0 / lam, used


@dataclass
class Trajectory:
    times: list = field(default_factory=list)
    a_c: list = field(default_factory=list)       # state after each step
    a_n: list = field(default_factory=list)       # recovered at each output
    iters: dict = field(default_factory=dict)
    maintenance: int = 0
    pcg_applies: int = 0
    steps: int = 0


def run(model: OracleModel, waveform, dt: float, n_steps: int, *,
        strategy="cspe", rel_tol=1e-8, max_iter=5000, max_cols=20, n_pod=10,
        eps_pod=1e-4, keep_states=True, a0=None) -> Trajectory:
    """schur.py:474-607 with a fixed dt, t_end = n_steps*dt and an output row
    after every step (output_period = dt*(1-1e-3)), i.e. 4 solves per step."""
    op = SchurOracle(model, waveform, strategy, rel_tol, max_iter, max_cols,
                     n_pod, eps_pod)
    t_end = n_steps * dt
    eps = 1e-12 * t_end
    a_c = np.zeros(model.n_c) if a0 is None else np.asarray(a0, float).copy()
    t = 0.0
    tr = Trajectory()
    a_n, _ = op.recover(a_c, t)
    if keep_states:
        tr.times.append(t)
        tr.a_c.append(a_c.copy())
        tr.a_n.append(a_n)
    steps = 0
    while t < t_end - eps:
        step_dt = min(dt, t_end - t)
        a_c, _ = op.euler(a_c, t, step_dt, steps + 1)
        t += step_dt
        steps += 1
        a_n, _ = op.recover(a_c, t)
        if keep_states:
            tr.times.append(t)
            tr.a_c.append(a_c.copy())
            tr.a_n.append(a_n)
    if not keep_states:
        tr.times.append(t)
        tr.a_c.append(a_c.copy())
        tr.a_n.append(a_n)
    tr.iters = {f: list(v) for f, v in op.iters.items()}
    tr.maintenance = op.strategy.maintenance
    tr.pcg_applies = op.pcg_applies
    tr.steps = steps
    return tr


def sinusoid(freq=50.0):
    """BASELINE configs' azimuthal coil current waveform sin(2 pi f t)."""
    w = 2.0 * np.pi * freq
    return lambda t: math.sin(w * t)
