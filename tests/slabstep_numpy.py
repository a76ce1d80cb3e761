"""CPU stand-in for a sharded-step slab (test infrastructure): the phase
methods of ``paper_1611_06721_b200.slabstep.SlabStepGrid`` on numpy arrays
(``csrc/solver_slab.cuh`` semantics: rank partials out, decisions on the
all-reduced totals), built on the oracle's blocks, so that ``SlabStepper``'s
host sequence and the ``torch.distributed`` communicator run under gloo on
CPU.  The CSPE decisions restate startvec.py:158-225 split at the
reductions, the conducting update schur.py:392-404 on the owned edges."""

from __future__ import annotations

import math

import numpy as np

from oracle import mq_oracle as O
from tests.slab_numpy import NumpySlab, edge_planes

NPART = 34


class NumpySlabStep(NumpySlab):
    def __init__(self, model, rank, world, *, max_cols=5, drop_tol=1e-8, strategy="cspe"):
        super().__init__(model, rank, world, O.jacobi_inverse(model.kn.diagonal())[0])
        self.m = model
        self.strategy = strategy
        self.max_cols, self.drop_tol = max_cols, drop_tol
        self.gidx = self.own
        self.n_n = self.own.size
        self.n_c = model.n_c
        _, ci, _ = edge_planes(model.shape, model.cond_global)
        self.owned = np.flatnonzero((ci >= self.lo) & (ci < self.hi)).astype(np.int64)
        self.n_own = self.owned.size
        for k in ("rhs_src", "rhs_cpl", "y_src", "y_cpl", "y_cur", "w1", "w2", "dvec"):
            self.V[k] = np.zeros_like(self.V["x"])
        self.vecs = {k: k for k in ("rhs_src", "rhs_cpl", "y_src", "y_cpl", "y_cur", "w2", "dvec")}
        self.a_c = np.zeros(self.n_c)
        # per family: own rows of U, K U (columns), replicated Galerkin G
        self.U = {f: np.zeros((self.n_n, 0)) for f in range(3)}
        self.KU = {f: np.zeros((self.n_n, 0)) for f in range(3)}
        self.G = {f: np.zeros((0, 0)) for f in range(3)}
        self.last = {}
        self._obs = {}
        self.minv = 1.0 / model.mc_diag

    # vectors named like the device ones
    def _y(self, fam):
        return {0: "y_src", 1: "y_cur", 2: "y_cpl"}[fam]

    def state_set(self, a_c):
        self.a_c = np.array(a_c, dtype=np.float64)

    def rhs(self, which, wave=0.0):
        if which == 0:
            self.V["rhs_src"][self.own_loc] = self.m.pattern[self.own] * wave
        else:
            self.V["rhs_cpl"][self.own_loc] = (self.m.kcn.T @ self.a_c)[self.own]

    def stage_b(self, which):
        self.V["b"][...] = self.V[which]

    def project(self, fam, which):
        part = np.zeros(NPART)
        if self.strategy != "cspe":
            return part
        rhs = self.own_values("rhs_src" if which == 0 else "rhs_cpl")
        k = self.U[fam].shape[1]
        part[:k] = self.U[fam].T @ rhs
        return part

    def start(self, fam, tot):
        x = np.zeros(self.n_n)
        if self.strategy == "cspe":
            beta = np.array(tot[: self.U[fam].shape[1]])
            while self.U[fam].shape[1]:
                try:
                    lo = O.chol_lower(self.G[fam])
                except O.PivotFail as bad:
                    keep = [i for i in range(self.U[fam].shape[1]) if i != bad.j]
                    self.U[fam], self.KU[fam] = self.U[fam][:, keep], self.KU[fam][:, keep]
                    self.G[fam] = self.G[fam][np.ix_(keep, keep)]
                    beta = beta[keep]
                    continue
                x = self.U[fam] @ O.chol_solve(lo, beta)
                break
        elif self.strategy == "previous" and fam in self.last:
            x = self.last[fam].copy()
        self.V["x"][...] = 0.0
        self.V["x"][self.own_loc] = x

    def store(self, fam, rep):
        self.V[self._y(fam)][self.own_loc] = self.own_values("x")

    def observe(self, fam, phase, tot=None):
        part = np.zeros(NPART)
        y = self.own_values(self._y(fam))
        if self.strategy == "previous":
            if phase == 0:
                self.last[fam] = y.copy()
            return part, 0
        U = self.U[fam]
        k = U.shape[1]
        st = self._obs.setdefault(fam, {})
        if phase == 0:
            part[:k] = U.T @ y
            part[k] = y @ y
        elif phase == 1:
            nv = math.sqrt(tot[k])
            st["nv"] = nv
            st["accept"] = not (nv == 0.0 or not math.isfinite(nv))
            if st["accept"]:
                w1 = y - U @ tot[:k]
                st["w1"] = w1
                part[:k] = U.T @ w1
                part[k] = w1 @ w1
        elif phase == 2:
            if st["accept"]:
                w2 = st["w1"] - U @ tot[:k]
                self.V["w2"][...] = 0.0
                self.V["w2"][self.own_loc] = w2
                part[0] = w2 @ w2
        elif phase == 3:
            if st["accept"]:
                nw = math.sqrt(tot[0])
                if nw < self.drop_tol * st["nv"]:
                    st["accept"] = False
                else:
                    st["nw"] = nw
                    if k == self.max_cols:   # FIFO eviction (startvec.py:180-184)
                        self.U[fam], self.KU[fam] = U[:, 1:], self.KU[fam][:, 1:]
                        self.G[fam] = self.G[fam][1:, 1:]
            return part, int(st["accept"])
        elif phase == 4:
            # u = w2 / ||w2|| and K u on own rows (w2's ghost planes refreshed)
            u_near = self._gather(self.V["w2"]) / st["nw"]
            u = u_near[self.own]
            ku = self.kn @ u_near
            st["u"], st["ku"] = u, ku
            kp = self.U[fam].shape[1]
            part[:kp] = self.U[fam].T @ ku
            part[kp] = u @ ku
        elif phase == 5:
            kp = self.U[fam].shape[1]
            g = np.empty((kp + 1, kp + 1))
            g[:kp, :kp] = self.G[fam]
            g[:kp, kp] = tot[:kp]
            g[kp, :kp] = tot[:kp]
            g[kp, kp] = tot[kp]
            self.G[fam] = g
            self.U[fam] = np.column_stack([self.U[fam], st["u"]])
            self.KU[fam] = np.column_stack([self.KU[fam], st["ku"]])
        return part, 0

    def euler_prep(self):
        self.V["dvec"][...] = 0.0
        self.V["dvec"][self.own_loc] = self.own_values("y_cpl") - self.own_values("y_src")

    def euler(self, dt):
        d = self._gather(self.V["dvec"])
        rate = (self.m.kcn[self.owned] @ d) - self.m.kc_apply(self.a_c, self.a_c)[self.owned]
        return self.a_c[self.owned] + dt * (self.minv[self.owned] * rate)

    def a_n_local(self):
        return self.own_values("y_src") - self.own_values("y_cur")

    def diagnostics(self):
        class D:
            pass
        d = D()
        d.basis_cols = [self.U[f].shape[1] for f in range(3)]
        d.columns_accepted = d.columns_dropped = d.evictions = d.solves = d.iterations = [0, 0, 0]
        d.maintenance_applies = d.pcg_applies = 0
        return d
