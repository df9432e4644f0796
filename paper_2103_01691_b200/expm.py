"""Matrix exponential on the GPU.

The reference takes every factor exponential on the host with scipy's Padé
scaling-and-squaring (linalg.py:59-72), and so does :func:`kron.prepare` by
default, as the north star asks.  The Magnus midpoint scheme, however, needs a
new exponential every step (problems.py:415-417), and on the host that
dominates the step for k >= ~64.  This module evaluates exp(A) on the device
with truncated Taylor series + scaling and squaring (the family the paper's
GPU code uses):

* s = max(0, ceil(log2 ||A||_1)) so that ||A / 2^s||_1 <= 1;
* degree-18 Taylor polynomial by Paterson–Stockmeyer (B^2, B^3, B^4, then
  Horner in B^4: 7 matrix products); the truncation remainder is bounded by
  ||B||^19 / 19! * 1.06 < 1e-17, below double-precision rounding;
* s squarings.

Every n x n matrix product is a μ-mode product through the C ABI (DMMA
kernels); the O(n^2) work (scaling, the Paterson–Stockmeyer block sums as one
(5 x 4) @ (4 x n^2) torch combination, the Horner additions) is torch
plumbing.  Diagonal inputs (the Magnus static factors) skip the series.  Results
agree with scipy.linalg.expm to ~1e-15 relative on the problems here
(tests/test_gpu_expm.py).
"""

from __future__ import annotations

import math

import numpy as np

from . import _device as dv
from . import _native
from .errors import InvalidInputError, ShapeError
from .kron import PropagatorCache

__all__ = ["DevicePropagatorCache", "matexp_device", "prepare_device"]

_DEGREE = 18
_COEF = [1.0 / math.factorial(k) for k in range(_DEGREE + 1)]


def _matmul(x, y):
    """Row-major n x n product x @ y as one μ-mode product (direction 2, n_left = n)."""
    n = x.shape[0]
    z = dv.torch.empty_like(x)
    code = dv.code(dv.np_dtype(x.dtype))
    _native.check(_native.lib().km_mumode(y.data_ptr(), code, x.data_ptr(), code, z.data_ptr(), n, n, n, 1,
                                          None, dv.stream_ptr(x.device)))
    return z


def matexp_device(a, dev=None, scale=1.0):
    """exp(scale * a) for a square matrix; returns a row-major device tensor (complex128 or float64).

    ``scale`` is applied on the device (and folded into the norm bound), so
    a host matrix is never rescaled on the host.
    """
    torch = dv.torch
    if dv.is_tensor(a):
        dev = a.device if a.is_cuda else (dev or dv.device())
        A = a.to(dev)
        norm1 = None
    else:
        a = np.asarray(a)
        if a.ndim != 2:
            raise ShapeError(f"matrix must be two-dimensional, got ndim={a.ndim}")
        dev = dev or dv.device()
        if a.shape[0] == a.shape[1] and a.size and np.count_nonzero(a) == np.count_nonzero(np.diagonal(a)):
            # diagonal: exp of the diagonal, no series (Magnus's static factors)
            diag = scale * np.diagonal(a).astype(np.result_type(a.dtype, np.float64))
            return dv.upload(np.diag(np.exp(diag)), dev)
        # the scaling exponent comes from the host copy: no device sync, so the
        # exponential queues behind (and overlaps) earlier device work
        norm1 = abs(scale) * float(np.abs(a).sum(axis=0).max()) if a.size else 0.0
        A = dv.upload(np.ascontiguousarray(a), dev)
    if A.dim() != 2 or A.shape[0] != A.shape[1]:
        raise ShapeError(f"matrix exponential needs a square matrix, got {tuple(A.shape)}")
    A = A.to(torch.complex128 if A.is_complex() else torch.float64).contiguous()
    n = A.shape[0]
    if norm1 is None:
        norm1 = abs(scale) * float(A.abs().sum(dim=0).max()) if n else 0.0
    if not math.isfinite(norm1):
        raise InvalidInputError("matrix exponential of non-finite entries")
    eye = torch.eye(n, dtype=A.dtype, device=dev)
    if norm1 == 0.0:
        return eye
    s = max(0, math.ceil(math.log2(norm1)))
    B = A * (scale * 2.0 ** -s)
    B2 = _matmul(B, B)
    B3 = _matmul(B2, B)
    B4 = _matmul(B2, B2)
    # the five Paterson-Stockmeyer blocks sum_i c[4j+i] B^i in ONE small
    # (5 x 4) @ (4 x n^2) combination instead of ~20 elementwise launches
    X = torch.stack((eye, B, B2, B3)).reshape(4, n * n)
    Q = (_ps_coefficients(A.dtype, dev) @ X).reshape(5, n, n)
    P = Q[4]
    for j in (3, 2, 1, 0):
        P = _matmul(P, B4).add_(Q[j])
    for _ in range(s):
        P = _matmul(P, P)
    return P


_PS_CACHE = {}


def _ps_coefficients(dtype, dev):
    key = (dtype, str(dev))
    hit = _PS_CACHE.get(key)
    if hit is None:
        c = _COEF
        rows = [[c[4 * j + i] for i in range(4)] for j in range(4)] + [[c[16], c[17], c[18], 0.0]]
        hit = _PS_CACHE[key] = dv.torch.tensor(rows, dtype=dtype, device=dev)
    return hit


class DevicePropagatorCache(PropagatorCache):
    """A :class:`PropagatorCache` whose factors were exponentiated on the device.

    ``exps`` (host arrays) is materialised lazily on first access; the device
    steps use the device factors directly.
    """

    def __init__(self, tau, dev_exps):
        object.__setattr__(self, "tau", tau)
        object.__setattr__(self, "_device", {})
        object.__setattr__(self, "_plans", {})  # kron.step's prebuilt calls (PropagatorCache._plans)
        object.__setattr__(self, "_dev_exps", tuple(dev_exps))
        object.__setattr__(self, "_host", None)

    @property
    def exps(self):
        if self._host is None:
            object.__setattr__(self, "_host", tuple(dv.to_host(e).copy() for e in self._dev_exps))
        return self._host

    @property
    def shape(self):
        return tuple(e.shape[0] for e in self._dev_exps)

    def exp_dtypes(self):
        return tuple(dv.np_dtype(e.dtype) for e in self._dev_exps)

    def device_exps(self, dtypes, dev):
        key = (tuple(np.dtype(t).str for t in dtypes), str(dev))
        hit = self._device.get(key)
        if hit is None:
            hit = tuple(e.to(device=dev, dtype=dv.torch_dtype(t)).contiguous() for e, t in zip(self._dev_exps, dtypes))
            self._device[key] = hit
        return hit

    def __repr__(self):
        return f"DevicePropagatorCache(tau={self.tau!r}, shape={self.shape})"


def prepare_device(op, tau, dev=None):
    """:func:`kron.prepare` with the exponentials taken on the GPU."""
    return DevicePropagatorCache(tau, tuple(matexp_device(np.asarray(a), dev, scale=tau) for a in op.factors))

