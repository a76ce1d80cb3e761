"""CPU stand-in for a GPU slab (test infrastructure): the same phase methods
as ``paper_1611_06721_b200.slab.SlabGrid`` on numpy arrays, with the oracle's
K_n, so ``slab_pcg_solve`` and ``TorchComm`` can run under gloo on CPU."""

from __future__ import annotations

import numpy as np

from paper_1611_06721_b200.slab import slab_range


def edge_planes(shape, gids):
    """(component, i, flat (j,k) plane index over (ny+1)(nz+1)) of global edge ids."""
    nx, ny, nz = shape
    n_ex = nx * (ny + 1) * (nz + 1)
    n_ey = (nx + 1) * ny * (nz + 1)
    comp = np.where(gids < n_ex, 0, np.where(gids < n_ex + n_ey, 1, 2))
    i = np.empty_like(gids); m = np.empty_like(gids)
    a = comp == 0
    q = gids[a]; i[a] = q // ((ny + 1) * (nz + 1)); r = q % ((ny + 1) * (nz + 1)); m[a] = r
    a = comp == 1
    q = gids[a] - n_ex; i[a] = q // (ny * (nz + 1)); r = q % (ny * (nz + 1))
    j, k = r // (nz + 1), r % (nz + 1); m[a] = j * (nz + 1) + k
    a = comp == 2
    q = gids[a] - n_ex - n_ey; i[a] = q // ((ny + 1) * nz); r = q % ((ny + 1) * nz)
    j, k = r // nz, r % nz; m[a] = j * (nz + 1) + k
    return comp, i, m


class NumpySlab:
    def __init__(self, model, rank, world, inv):
        import torch
        self.torch = torch
        nx, ny, nz = model.shape
        self.lo, self.hi = slab_range(nx, world, rank)
        self.n_planes = self.hi - self.lo
        self.inv = inv
        g = model.noncond_global
        comp, i, m = edge_planes(model.shape, g)
        self.own = np.flatnonzero((i >= self.lo) & (i < self.hi))
        near = np.flatnonzero((i >= self.lo - 1) & (i <= self.hi))
        self.near = near
        self.loc = (comp[near], i[near] - self.lo + 1, m[near])  # plane index 0 = ghost lo
        own_pos = np.searchsorted(near, self.own)
        self.own_loc = tuple(a[own_pos] for a in self.loc)
        self.kn = model.kn[self.own]
        self.n_glob = model.n_n
        shape = (3, self.n_planes + 2, (ny + 1) * (nz + 1))
        self.V = {k: np.zeros(shape) for k in ("x", "b", "r", "pa", "pb", "ap")}

    def set_global(self, name, vec):
        self.V[name][...] = 0.0
        self.V[name][self.own_loc] = vec[self.own]

    def own_values(self, name):
        return self.V[name][self.own_loc]

    def _gather(self, arr):
        xg = np.zeros(self.n_glob)
        xg[self.near] = arr[self.loc]
        return xg

    def plane_views(self, name, plane):
        return [self.torch.from_numpy(self.V[name][c, plane + 1]) for c in range(3)]

    def send_planes(self, name):
        return {"lo": self.plane_views(name, 0), "hi": self.plane_views(name, self.n_planes - 1)}

    def ghost_planes(self, name):
        return {"lo": self.plane_views(name, -1), "hi": self.plane_views(name, self.n_planes)}

    def init(self, x0_mode, jac):
        b = self.own_values("b")
        if x0_mode == 1:
            r = b - self.kn @ self._gather(self.V["x"])
        else:
            self.V["x"][self.own_loc] = 0.0
            r = b.copy()
        self.V["r"][self.own_loc] = r
        z = self.inv * r if jac else r
        return np.array([b @ b, r @ r, r @ z])

    def k1(self, first, beta, alpha_prev, pold_is_a, jac):
        pold = self.V["pa" if pold_is_a else "pb"]
        pnew = self.V["pb" if pold_is_a else "pa"]
        r = self.V["r"]
        z = self.inv * r if jac else r
        pn_all = z if first else z + beta * pold
        if not first:
            self.V["x"][self.own_loc] = self.V["x"][self.own_loc] + alpha_prev * pold[self.own_loc]
        pnew[self.own_loc] = pn_all[self.own_loc]
        ap = self.kn @ self._gather(pn_all)
        self.V["ap"][self.own_loc] = ap
        return np.array([pn_all[self.own_loc] @ ap])

    def k2(self, alpha, jac):
        r = self.V["r"][self.own_loc] - alpha * self.V["ap"][self.own_loc]
        self.V["r"][self.own_loc] = r
        z = self.inv * r if jac else r
        return np.array([r @ r, r @ z])

    def final(self, alpha, p_is_a):
        p = self.V["pa" if p_is_a else "pb"]
        self.V["x"][self.own_loc] = self.V["x"][self.own_loc] + alpha * p[self.own_loc]
