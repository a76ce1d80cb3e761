"""Per-step A-field parity at config scale (test infrastructure).

The north-star bar is the relative L2 error of the whole A-field — the
concatenation (a_c, a_n) in the reference's compact order — at every time
step.  Storing every oracle state at 64^3 / 128^3 is 6 / 49 MB per step, so
the fixtures hold, per step, the exact norm ``||A_ref||`` and a CountSketch
``S A_ref`` (M buckets, bucket and sign of every entry from a seeded
generator).  ``S`` is linear, so ``||S A_gpu - S A_ref|| = ||S (A_gpu -
A_ref)||``, an unbiased estimate of ``||A_gpu - A_ref||`` whose relative
standard deviation is about ``sqrt(2/M)`` (2.2 % at M = 4096).  The final
step of every fixture also stores the full field, so the tests check the
estimate against the exact error there.
"""

from __future__ import annotations

import numpy as np

SKETCH_M = 4096
SKETCH_SEED = 1611_06721


def sketch_plan(n: int, m: int = SKETCH_M, seed: int = SKETCH_SEED):
    """Bucket and sign of every entry of an n-long field (deterministic)."""
    rng = np.random.default_rng([seed, n])
    bucket = rng.integers(0, m, n, dtype=np.int64)
    sign = rng.integers(0, 2, n, dtype=np.int8).astype(np.float64) * 2.0 - 1.0
    return bucket, sign


def sketch(field: np.ndarray, plan, m: int = SKETCH_M) -> np.ndarray:
    bucket, sign = plan
    return np.bincount(bucket, weights=sign * np.asarray(field, np.float64), minlength=m)


def field_of(a_c, a_n) -> np.ndarray:
    return np.concatenate([np.asarray(a_c, np.float64), np.asarray(a_n, np.float64)])


def sketched_rel(field_gpu, sk_ref, norm_ref, plan) -> float:
    """Estimated ||A_gpu - A_ref|| / ||A_ref|| from the reference's sketch."""
    d = sketch(field_gpu, plan, sk_ref.shape[-1]) - sk_ref
    return float(np.linalg.norm(d) / (norm_ref if norm_ref > 0 else 1.0))


def exact_rel(field_gpu, field_ref) -> float:
    nb = np.linalg.norm(field_ref)
    return float(np.linalg.norm(np.asarray(field_gpu) - field_ref) / (nb if nb > 0 else 1.0))
