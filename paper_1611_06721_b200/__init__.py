"""mq-b200: B200-native drop-in for the hot path of arXiv 1611.06721 (``mqsolve``).

The repeated PCG pseudo-inverse solve on the singular nonconducting curl-curl
block, its SPE/CSPE and POD start vectors, the Brauer K_c update and the
explicit-Euler update, as hand-written sm_100a kernels behind the C ABI of
``libmq_b200.so`` (``include/mq_b200.h``), with the reference's Python entry
points mirrored here.
"""

from .device import AIR, COIL, CONDUCTOR, NU_VACUUM, DeviceGrid, KnOperator, Problem, sinusoid
from .krylov import (IndefiniteOperatorError, JacobiPreconditioner, PcgConfig, Preconditioner,
                     SolveReport, pcg_solve)
from .schur import (FAMILIES, CflEstimate, SchurOperator, StepFailureError, TransientResult,
                    estimate_cfl, explicit_euler_step, recover_an, run_explicit, trace_bytes)
from .startvec import DeviceStrategy, RhsFamily

__version__ = "0.1.0"

__all__ = [
    "AIR", "COIL", "CONDUCTOR", "NU_VACUUM", "DeviceGrid", "KnOperator", "Problem", "sinusoid",
    "IndefiniteOperatorError", "JacobiPreconditioner", "PcgConfig", "Preconditioner",
    "SolveReport", "pcg_solve", "FAMILIES", "SchurOperator", "StepFailureError",
    "TransientResult", "explicit_euler_step", "recover_an", "run_explicit", "DeviceStrategy",
    "CflEstimate", "estimate_cfl", "trace_bytes",
    "RhsFamily",
]
