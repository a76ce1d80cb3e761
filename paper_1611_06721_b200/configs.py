"""BASELINE.json workloads as :class:`~paper_1611_06721_b200.device.Problem`s.

The reference ships no geometry for these configs (its ``builtin_model`` is a
single bar with one loop, model.py:582-628), so the recipe of SURVEY.md
section 8(d) is applied, identically for the device path and the oracle:

* unit cube, N^3 cells, h = 1/N; iron blocks of CONDUCTOR cells; air nu0;
* the annular coil is a stack of closed square node loops (model.py:158-180
  semantics per loop) of half-widths 4N/16..6N/16 around the z axis in the
  4N/16+1 central node planes, each loop carrying J*h^2 ampere-turns; COIL
  cells (cosmetic, COIL == air for nu) mark the annulus;
* waveform sin(2 pi 50 t).

Config 2 and 4 carry two disjoint iron blocks, which the reference's
``assemble`` rejects (model.py:428-435); the device path has no such check.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .device import AIR, COIL, CONDUCTOR, NU_VACUUM, Problem, sinusoid


@dataclass(frozen=True)
class LoopSpec:
    i0: int
    i1: int
    j0: int
    j1: int
    k0: int
    amps: float


@dataclass
class ConfigSpec:
    name: str
    N: int
    blocks: list            # [(i0,i1,j0,j1,k0,k1)] conductor cell boxes
    kappa: float
    brauer: tuple
    J: float
    steps: int
    strategy: str
    max_cols: int = 5
    n_pod: int = 20
    freq: float = 50.0
    rel_tol: float = 1e-8
    max_iter: int = 5000
    dt: float | None = None  # measured 0.9*CFL when known

    @property
    def h(self) -> float:
        return 1.0 / self.N


LINEAR_IRON = (0.0, 0.0, NU_VACUUM / 1000.0)
BRAUER_IRON = (3.8, 2.17, 396.2)


def coil_loops(N: int, J: float) -> list[LoopSpec]:
    s = N // 16
    c = N // 2
    h = 1.0 / N
    amps = J * h * h
    loops = []
    for k0 in range(c - 2 * s, c + 2 * s + 1):
        for w in range(4 * s, 6 * s + 1):
            loops.append(LoopSpec(c - w, c + w, c - w, c + w, k0, amps))
    return loops


def material_map(spec: ConfigSpec) -> np.ndarray:
    N = spec.N
    mat = np.zeros((N, N, N), dtype=np.int8)
    s, c = N // 16, N / 2
    ctr = np.arange(N) + 0.5
    r = np.maximum(np.abs(ctr[:, None] - c), np.abs(ctr[None, :] - c))
    ring = (r >= 4 * s) & (r <= 6 * s)
    kz = slice(N // 2 - 2 * s, N // 2 + 2 * s)
    mat[:, :, kz][ring] = COIL
    for (i0, i1, j0, j1, k0, k1) in spec.blocks:
        mat[i0:i1, j0:j1, k0:k1] = CONDUCTOR
    return mat


def config_spec(index: int) -> ConfigSpec:
    if index == 0:
        return ConfigSpec("cfg0_16cube_linear_cspe5", 16, [(5, 11, 5, 11, 5, 11)], 5e6,
                          LINEAR_IRON, 1e6, 100, "cspe", max_cols=5, dt=3.603515e-3)
    if index in (1, 3):
        return ConfigSpec("cfg1_64cube_brauer_cspe5" if index == 1 else "cfg3_64cube_ensemble",
                          64, [(20, 44, 20, 44, 20, 44)], 5e6, BRAUER_IRON, 5e6,
                          400 if index == 1 else 200, "cspe", max_cols=5, n_pod=20,
                          dt=2.256829e-4)
    if index == 2:
        c = 64
        return ConfigSpec("cfg2_128cube_two_blocks_pod30", 128,
                          [(c - 28, c - 4, c - 12, c + 12, c - 12, c + 12),
                           (c + 4, c + 28, c - 12, c + 12, c - 12, c + 12)],
                          5e6, BRAUER_IRON, 5e6, 200, "pod", n_pod=30,
                          dt=5.641670141705834e-05)  # device estimate_cfl, safety 0.9
    if index == 4:
        c = 128
        return ConfigSpec("cfg4_256cube_two_blocks_cspe5", 256,
                          [(c - 56, c - 8, c - 24, c + 24, c - 24, c + 24),
                           (c + 8, c + 56, c - 24, c + 24, c - 24, c + 24)],
                          5e6, BRAUER_IRON, 5e6, 50, "cspe", max_cols=5,
                          dt=1.4106248992090958e-05)  # device estimate_cfl, safety 0.9
    raise ValueError(f"unknown config {index}")


# ---- host-side partition for building the compact source pattern ----------

def noncond_positions(material: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """(is_noncond over global edge ids, compact index over global ids or -1).

    Same rules as the device context (model.py:240-272, 455-462)."""
    nx, ny, nz = material.shape
    cond = np.pad(material == CONDUCTOR, 1)
    out = []
    for comp in range(3):
        shp = [nx + 1, ny + 1, nz + 1]
        shp[comp] -= 1
        bnd = np.zeros(shp, dtype=bool)
        for ax in range(3):
            if ax == comp:
                continue
            idx = [slice(None)] * 3
            idx[ax] = [0, shp[ax] - 1]
            bnd[tuple(idx)] = True
        # four cells around the edge, in padded cell coordinates
        a, b = [d for d in range(3) if d != comp]
        touch = np.zeros(shp, dtype=bool)
        for da in (0, 1):
            for db in (0, 1):
                sl = [None] * 3
                sl[comp] = slice(1, 1 + shp[comp])
                sl[a] = slice(da, da + shp[a])
                sl[b] = slice(db, db + shp[b])
                touch |= cond[tuple(sl)]
        out.append((~bnd & ~touch).reshape(-1))
    flag = np.concatenate(out)
    idx = np.cumsum(flag) - 1
    idx[~flag] = -1
    return flag, idx


def loop_edges(shape, lp: LoopSpec):
    """Global edge ids and signs of a rectangular loop (model.py:321-336)."""
    nx, ny, nz = shape
    n_ex = nx * (ny + 1) * (nz + 1)

    def ex(i, j, k):
        return (np.asarray(i) * (ny + 1) + j) * (nz + 1) + k

    def ey(i, j, k):
        return n_ex + (i * ny + np.asarray(j)) * (nz + 1) + k

    ii = np.arange(lp.i0, lp.i1)
    jj = np.arange(lp.j0, lp.j1)
    ids = np.concatenate([ex(ii, lp.j0, lp.k0), ey(lp.i1, jj, lp.k0),
                          ex(ii, lp.j1, lp.k0), ey(lp.i0, jj, lp.k0)])
    sg = np.concatenate([np.ones(ii.size), np.ones(jj.size), -np.ones(ii.size), -np.ones(jj.size)])
    return ids, sg


def source_pattern(material: np.ndarray, loops) -> np.ndarray:
    """Sum of the loops' compact patterns (model.py:552-556 per loop)."""
    flag, idx = noncond_positions(material)
    n_n = int(flag.sum())
    pattern = np.zeros(n_n)
    touched = np.zeros(n_n, dtype=np.int32)
    for lp in loops:
        ids, sg = loop_edges(material.shape, lp)
        pos = idx[ids]
        if (pos < 0).any():
            raise ValueError("coil loop touches boundary or conducting edges")
        # one closed loop visits an edge at most once
        pattern[pos] += sg * lp.amps
        touched[pos] += 1
    # edge-disjoint loops: every entry is a single term, so the in-place
    # accumulation equals the reference shim's pattern + one per loop bitwise
    if touched.max(initial=0) > 1:
        raise ValueError("coil loops share edges")
    return pattern


def make_problem(index: int, *, j_scale: float = 1.0, kappa_scale: float = 1.0) -> Problem:
    spec = config_spec(index)
    mat = material_map(spec)
    loops = coil_loops(spec.N, spec.J * j_scale)
    return Problem(material=mat, h=spec.h, kappa=spec.kappa * kappa_scale, brauer=spec.brauer,
                   nu_air=NU_VACUUM, pattern=source_pattern(mat, loops),
                   waveform=sinusoid(spec.freq), name=spec.name,
                   meta={"spec": spec, "loops": loops})


def builtin_problem(cells: int = 8, h: float = 5e-3, kappa: float = 5e6,
                    brauer: tuple = (49.4, 1.46, 520.6), amps: float = 50000.0, tau: float = 0.5, *,
                    linear: bool = False) -> Problem:
    """The reference's benchmark model (model.py:582-622) as a Problem: a
    2 x 2 x (cells - 2) conductor bar at the grid centre, threaded by one
    square edge loop one cell in from the boundary at mid height, carrying
    ``amps`` with the exponential ramp 1 - exp(-t/tau); COIL cells mark the
    two cell layers around the loop; ``linear`` freezes the bar reluctivity
    at its unsaturated value k1 + k3."""
    import math
    if cells < 6:
        raise ValueError("builtin model needs at least 6 cells per direction")
    n = int(cells)
    mat = np.zeros((n, n, n), dtype=np.int8)
    b0, b1 = n // 2 - 1, n // 2
    mat[b0:b1 + 1, b0:b1 + 1, 1:n - 1] = CONDUCTOR
    lp = LoopSpec(1, n - 1, 1, n - 1, n // 2, float(amps))
    coil = np.zeros((n, n, n), dtype=bool)
    for kk in (lp.k0 - 1, lp.k0):
        if 0 <= kk < n:
            coil[lp.i0:lp.i1, lp.j0 - 1:lp.j0 + 1, kk] = True
            coil[lp.i0:lp.i1, lp.j1 - 1:lp.j1 + 1, kk] = True
            coil[lp.i0 - 1:lp.i0 + 1, lp.j0:lp.j1, kk] = True
            coil[lp.i1 - 1:lp.i1 + 1, lp.j0:lp.j1, kk] = True
    mat[coil & (mat == AIR)] = COIL
    k1, k2, k3 = (float(v) for v in brauer)
    nu = (0.0, 0.0, k1 + k3) if linear else (k1, k2, k3)
    tau = float(tau)
    return Problem(material=mat, h=float(h), kappa=float(kappa), brauer=nu, nu_air=NU_VACUUM,
                   pattern=source_pattern(mat, [lp]), waveform=lambda t: 1.0 - math.exp(-t / tau),
                   name=f"builtin_{n}", meta={"loops": [lp], "linear": bool(linear)})


def ensemble_factors(n_members: int = 256, seed: int = 0):
    """Config 3: J then kappa factors, each U(0.8, 1.2)."""
    rng = np.random.default_rng(seed)
    j = rng.uniform(0.8, 1.2, n_members)
    k = rng.uniform(0.8, 1.2, n_members)
    return j, k
