"""Small dense helpers on the host: the factor exponential, products, solves, norms.

The north star keeps E_mu = exp(tau*A_mu) as small host-precomputed n x n
inputs, as the reference does (linalg.py:59-72 → scipy.linalg.expm,
Al-Mohy–Higham Padé).  Argument checks raise the reference's exception types
with its messages (linalg.py:23-56), so callers that match on them keep
working; the GPU never sees these O(n^3) n x n operations.
"""

from __future__ import annotations

import numpy as np
import scipy.linalg

from .errors import InvalidInputError, ShapeError, SingularMatrixError

try:
    from threadpoolctl import threadpool_limits
except ImportError:  # pragma: no cover
    threadpool_limits = None

__all__ = ["matexp", "matmul", "one_norm", "solve"]

# factors up to this size are exponentiated on one BLAS thread: threading does
# not pay there, and many small exponentials then do not fight over the pool
_ONE_THREAD_MAX = 256


def _two_d(x, label):
    x = np.asarray(x)
    if x.ndim == 2:
        return x
    raise ShapeError(f"{label} must be two-dimensional, got ndim={x.ndim}")


def matexp(a):
    """exp(a) by scipy's scaling-and-squaring Padé; a real ``a`` gives a real result, exp(0) = I."""
    a = _two_d(a, "matrix")
    rows, cols = a.shape
    if rows != cols:
        raise ShapeError(f"matrix exponential needs a square matrix, got {a.shape}")
    if not np.isfinite(a).all():
        raise InvalidInputError("matrix exponential of non-finite entries")
    if threadpool_limits is None or rows > _ONE_THREAD_MAX:
        return scipy.linalg.expm(a)
    with threadpool_limits(limits=1):
        return scipy.linalg.expm(a)


def one_norm(a):
    """max_j sum_i |a_ij|."""
    col_sums = np.abs(_two_d(a, "matrix")).sum(axis=0)
    return float(col_sums.max())


def matmul(a, b):
    """a @ b, refusing mismatched inner extents."""
    lhs, rhs = _two_d(a, "left operand"), _two_d(b, "right operand")
    if lhs.shape[1] == rhs.shape[0]:
        return lhs @ rhs
    raise ShapeError(f"cannot multiply {lhs.shape} by {rhs.shape}")


def solve(a, b):
    """x with a @ x = b (LAPACK LU with partial pivoting); singular a raises SingularMatrixError."""
    coef = _two_d(a, "coefficient matrix")
    if coef.shape[0] != coef.shape[1]:
        raise ShapeError(f"coefficient matrix must be square, got {coef.shape}")
    rhs = np.asarray(b)
    if rhs.ndim not in (1, 2) or rhs.shape[0] != coef.shape[0]:
        raise ShapeError(f"right-hand side of shape {rhs.shape} does not match {coef.shape}")
    try:
        return np.linalg.solve(coef, rhs)
    except np.linalg.LinAlgError as exc:
        raise SingularMatrixError(f"linear solve failed: {exc}") from exc
