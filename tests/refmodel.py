"""The reference's own model of a BASELINE config (test infrastructure).

Builds a config with the REFERENCE's ``assemble`` plus the SURVEY.md 8(d)
shim (sum of closed coil loops, sinusoidal waveform, the connectivity check
bypassed for two blocks), from whichever ``mqsolve`` is importable: the
read-only tree in the build container, or the copy installed into
``baseline/_ref`` that travels to the GPU box.  Used by
tests/golden/make_golden*.py and the reference-binding GPU tests.
"""

from __future__ import annotations

import math

import numpy as np

from paper_1611_06721_b200 import configs as C


def reference_model(index: int, brauer=None):
    """Reference assemble + the SURVEY 8(d) shim (sum of loops, sin waveform)."""
    import mqsolve.model as M
    from mqsolve import Excitation, GridSpec, Material, ScaledPatternSource
    spec = C.config_spec(index)
    mat = C.material_map(spec)
    loops = C.coil_loops(spec.N, spec.J)
    k1, k2, k3 = brauer or spec.brauer
    cond = Material(kappa=spec.kappa, brauer_k1=k1, brauer_k2=k2, brauer_k3=k3)
    first = loops[0]
    exc = Excitation(first.i0, first.i1, first.j0, first.j1, first.k0, amps=first.amps)
    grid = GridSpec(spec.N, spec.N, spec.N, spec.h, mat)
    saved = M._check_conductor_region
    M._check_conductor_region = lambda mask: None   # two disjoint blocks (configs 2, 4)
    try:
        model = M.assemble(grid, cond, exc)
    finally:
        M._check_conductor_region = saved
    topo = M._Topology(grid)
    interior = model.interior_edges
    pos = np.full(topo.n_edges, -1, dtype=np.int64)
    pos[interior] = np.arange(interior.size)
    nidx = np.full(interior.size, -1, dtype=np.int64)
    nidx[model.nonconducting] = np.arange(model.nonconducting.size)
    pattern = np.zeros(model.n_n)
    for lp in loops:
        ids, sg = topo.loop_edges(Excitation(lp.i0, lp.i1, lp.j0, lp.j1, lp.k0, amps=lp.amps))
        one = np.zeros(model.n_n)
        np.add.at(one, nidx[pos[ids]], sg * lp.amps)
        pattern = pattern + one
    w = 2.0 * np.pi * spec.freq
    model.system.source = ScaledPatternSource(pattern, lambda t: math.sin(w * t))
    return spec, model, pattern
