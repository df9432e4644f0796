"""Host-side matrix exponential for the 1D factors.

The north star keeps E_mu = exp(tau*A_mu) as small host-precomputed n x n
inputs, exactly as the reference does (linalg.py:59-72 → scipy.linalg.expm,
Al-Mohy–Higham Padé).  Same checks and messages as the reference.
"""

from __future__ import annotations

import numpy as np
import scipy.linalg

from .errors import InvalidInputError, ShapeError

try:
    from threadpoolctl import threadpool_limits
except ImportError:  # pragma: no cover
    threadpool_limits = None

__all__ = ["matexp"]

# below this size BLAS threading gains nothing for the exponential (linalg.py:17-20)
_SINGLE_THREAD_EXP_DIM = 256


def matexp(a):
    """Matrix exponential by diagonal Padé approximation with scaling and squaring.

    Real input yields real output; ``matexp(0) == I`` exactly.
    """
    a = np.asarray(a)
    if a.ndim != 2:
        raise ShapeError(f"matrix must be two-dimensional, got ndim={a.ndim}")
    if a.shape[0] != a.shape[1]:
        raise ShapeError(f"matrix exponential needs a square matrix, got {a.shape}")
    if not np.isfinite(a).all():
        raise InvalidInputError("matrix exponential of non-finite entries")
    if threadpool_limits is not None and a.shape[0] <= _SINGLE_THREAD_EXP_DIM:
        with threadpool_limits(limits=1):
            return scipy.linalg.expm(a)
    return scipy.linalg.expm(a)
