"""numpy restatement of the reference's hot path (kronmode 0.1.0) — TEST INFRASTRUCTURE.

This module is the checker the GPU path is compared against and the CPU
baseline ``bench.py`` times; the product never imports it (see
oracle/__init__.py).  Each function restates one reference function with the
same numpy/BLAS calls in the same order, so that (a) its results agree with
the reference bit for bit on the same BLAS, and (b) its run time is the
reference's run time.  Pinning: tests/test_oracle_golden.py checks every
function below against golden vectors produced by the reference itself
(tests/golden/make_golden.py imports /root/reference/pkg/src in the dev
container and writes tests/golden/*.npz).

Reference anchors (files under /root/reference/pkg/src/kronmode):
  mu_mode_product      tensor.py:80-140
  tucker               tensor.py:143-166
  step                 kron.py:110-121
  forward_transform    hermite.py:108-121
  inverse_transform    hermite.py:124-142
  weight_product       problems.py:528-539
  nonlinear_half       problems.py:542-545
  gpe_strang_step      problems.py:548-565
  tdpot_strang_step    restated from primitives
  magnus step loop     problems.py:397-420
"""

from __future__ import annotations

from math import prod

import numpy as np


def mu_mode_product(u, mat, mu):
    """tensor.py:80-140: mode 1 is one GEMM on the unfolding, others a loop of slab GEMMs."""
    u = np.asarray(u)
    mat = np.asarray(mat)
    ax = mu - 1
    shp = u.shape
    n_mu = shp[ax]
    m = mat.shape[0]
    assert mat.shape[1] == n_mu
    out_dtype = np.result_type(u.dtype, mat.dtype)
    uf = u if u.flags.f_contiguous else np.asfortranarray(u)
    if uf.dtype != out_dtype:
        uf = uf.astype(out_dtype, order="F")
    if mat.dtype != out_dtype:
        mat = mat.astype(out_dtype)
    out_shape = shp[:ax] + (m,) + shp[ax + 1:]
    if ax == 0:
        unfold = uf.reshape((n_mu, -1), order="F")
        return np.matmul(unfold.T, mat.T).T.reshape(out_shape, order="F")
    n_left = prod(shp[:ax])
    n_right = prod(shp[ax + 1:])
    cube = uf.reshape((n_left, n_mu, n_right), order="F")
    out = np.empty((n_left, m, n_right), dtype=out_dtype, order="F")
    for r in range(n_right):
        np.matmul(mat, cube[:, :, r].T, out=out[:, :, r].T)
    return out.reshape(out_shape, order="F")


def tucker(u, mats):
    """tensor.py:143-166: ascending directions, None skipped."""
    out = np.asarray(u)
    for mu, mat in enumerate(mats, start=1):
        if mat is not None:
            out = mu_mode_product(out, mat, mu)
    return out


def step(exps, u):
    """kron.py:110-121: tucker with the cached exponentials."""
    return tucker(u, list(exps))


def forward_transform(phis, weights, values):
    """hermite.py:108-121: weight broadcast per direction, then tucker(phi)."""
    values = np.asarray(values)
    d = values.ndim
    weighted = values
    for ax, w in enumerate(weights):
        shape = (1,) * ax + (w.size,) + (1,) * (d - ax - 1)
        weighted = weighted * np.asarray(w).reshape(shape)
    return tucker(weighted, list(phis))


def inverse_transform(mats, coeffs):
    """hermite.py:124-142: tucker with phi^H (or the q x k evaluation matrices)."""
    return tucker(coeffs, list(mats))


def weight_product(weights, shape):
    """problems.py:528-539."""
    d = len(shape)
    out = np.ones(shape, order="F")
    for ax, w in enumerate(weights):
        w = np.asarray(w, dtype=float)
        out *= w.reshape((1,) * ax + (w.size,) + (1,) * (d - ax - 1))
    return out


def nonlinear_half(psi, weight_prod, half_tau):
    """problems.py:542-545."""
    density = (psi.real**2 + psi.imag**2) / weight_prod
    return psi * np.exp((0.5j * half_tau) * (1.0 - density))


def gpe_strang_step(exps, weights, psi, tau):
    """problems.py:548-565."""
    psi = np.asarray(psi)
    wp = weight_product(weights, psi.shape)
    psi = nonlinear_half(psi, wp, 0.5 * tau)
    psi = step(exps, psi)
    return nonlinear_half(psi, wp, 0.5 * tau)


def sin2_integral(t_a, t_b):
    import math

    return (t_b / 2 - math.sin(2 * t_b) / 4) - (t_a / 2 - math.sin(2 * t_a) / 4)


def tdpot_strang_step(exps, x_nodes, psi, t, tau, direction=3):
    """Configuration 4: exact potential phase / exact linear step / phase.

    Composed only of reference primitives (``step``) plus a numpy phase, in
    the structure of problems.py:548-565.
    """
    psi = np.asarray(psi)
    d = psi.ndim
    shape = (1,) * (direction - 1) + (psi.shape[direction - 1],) + (1,) * (d - direction)
    x = np.asarray(x_nodes, dtype=float)
    f_a = np.exp(-1j * x * sin2_integral(t, t + 0.5 * tau)).reshape(shape)
    f_b = np.exp(-1j * x * sin2_integral(t + 0.5 * tau, t + tau)).reshape(shape)
    psi = psi * f_a
    psi = step(exps, psi)
    return psi * f_b


def magnus_propagate(coeffs0, exp_static, driven_exps):
    """problems.py:413-420: per-step tucker(coeffs, (E_s, E_s, E_driven(t_mid)))."""
    coeffs = coeffs0
    for e_dr in driven_exps:
        coeffs = tucker(coeffs, (exp_static, exp_static, e_dr))
    return coeffs


def rel_l2(a, b):
    """Relative l2 error ||a - b|| / ||b|| (the north star's parity metric)."""
    a = np.asarray(a)
    b = np.asarray(b)
    den = np.linalg.norm(b.ravel())
    return float(np.linalg.norm((a - b).ravel()) / (den if den else 1.0))
