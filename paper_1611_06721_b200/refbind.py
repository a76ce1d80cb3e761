"""Glue that plugs the device path into the reference's own entry points.

INTEGRATION.md sections 1-2 as code, so that the bindings a maintainer of
``mqsolve`` would add are the ones the tests run:

* :func:`bind_pcg` rebinds the module-global ``pcg_solve`` of
  ``mqsolve.schur`` (imported at mq/schur.py:32-33 and called by
  ``SchurOperator.solve_kn`` :253 and ``apply_detached`` :307).  Every solve
  on a ``_CountedApply`` -- the K_n operator a ``SchurOperator`` hands to
  ``pcg_solve`` (mq/schur.py:156-166,191) -- runs as one fused device PCG on
  the matrix-free K_n of a :class:`~paper_1611_06721_b200.device.DeviceGrid`;
  the operator's application counter advances by the device's count, so
  ``pcg_applies`` and the aggregates stay the reference's.  Any other operator
  (e.g. a consistent-mass M_c solve, mq/schur.py:280-287) goes to the
  reference's own ``pcg_solve``.
* :func:`device_strategy` builds a device start-vector strategy that is an
  instance of the reference's ``StartVectorStrategy`` class, as
  ``SchurOperator(strategy=...)`` / ``run_explicit(strategy=...)`` require
  (mq/schur.py:198-199 tests ``isinstance``, not the protocol).

Nothing here imports the reference: the caller passes its modules in.
"""

from __future__ import annotations

from .device import DeviceGrid, Problem
from .krylov import pcg_solve as _device_pcg
from .startvec import DeviceStrategy

__all__ = ["PcgBinding", "bind_pcg", "device_strategy", "grid_for_model"]


def grid_for_model(model, device: int = 0) -> DeviceGrid:
    """A device context for a reference ``Model`` (mq/model.py:438-518)."""
    return DeviceGrid(Problem.from_reference_model(model), device)


class PcgBinding:
    """Callable with the reference's ``pcg_solve`` signature (mq/krylov.py:174)."""

    def __init__(self, schur_module, grid: DeviceGrid):
        self.S = schur_module
        self.grid = grid
        self.kn = grid.kn_operator()
        self.reference_pcg = schur_module.pcg_solve
        self.device_solves = 0

    def __call__(self, a, b, x0=None, config=None, preconditioner=None):
        if type(a).__name__ == "_CountedApply":
            x, rep = _device_pcg(self.kn, b, x0=x0, config=config, preconditioner=preconditioner)
            a.count += rep.applications
            self.device_solves += 1
            return x, self.S.SolveReport(rep.iterations, rep.final_rel_residual, rep.converged)
        return self.reference_pcg(a, b, x0, config, preconditioner)

    def __enter__(self):
        self.S.pcg_solve = self
        return self

    def __exit__(self, *exc):
        self.S.pcg_solve = self.reference_pcg
        return False


def bind_pcg(schur_module, grid: DeviceGrid) -> PcgBinding:
    """Rebind ``schur_module.pcg_solve``; use as a context manager to restore it."""
    return PcgBinding(schur_module, grid)


def device_strategy(grid: DeviceGrid, kind: str = "cspe", base=None, **kw) -> DeviceStrategy:
    """A device strategy the reference accepts as ``strategy=``.

    ``SchurOperator`` takes an instance only if it IS a
    ``mqsolve.startvec.StartVectorStrategy`` (``isinstance`` check,
    mq/schur.py:198-199; anything else goes to ``make_strategy`` as a name), so
    pass that class as ``base``: the returned object is an instance of a
    subclass of both, whose protocol methods (mq/startvec.py:315-342) are the
    device ones.  Without ``base`` a plain :class:`DeviceStrategy` is returned
    (for this package's own ``SchurOperator``)."""
    if base is None:
        return DeviceStrategy(grid, kind, **kw)
    cls = _DEVICE_SUBCLASSES.get(base)
    if cls is None:
        cls = type("DeviceStartVectorStrategy", (DeviceStrategy, base), {"__module__": __name__})
        _DEVICE_SUBCLASSES[base] = cls
    return cls(grid, kind, **kw)


_DEVICE_SUBCLASSES: dict = {}
