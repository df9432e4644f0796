"""Splitting and Magnus compositions on the GPU, plus the host setup they need.

Drop-in for the hot-path part of the reference's ``kronmode.problems``:

* :func:`gpe_strang_step` (problems.py:548-565): half nonlinear phase, exact
  linear step, half nonlinear phase.  One ``km_tucker`` call: the first phase
  is a standalone pass, the d products run on DMMA and the second phase is
  fused into the epilogue of the last product; the weight product
  (problems.py:528-539, rebuilt every step there) is formed in registers from
  the d weight vectors.
* :func:`tdpot_strang_step` — the configuration-4 scheme (no reference
  driver; restated from reference primitives in SURVEY §8(c)): Strang
  splitting of ``i psi' = H psi + x_3 sin(t)^2 psi`` with the exactly
  integrated potential phase ``exp(-i x_3 ∫ sin^2)`` fused into the same
  prologue/epilogue slots.
* :func:`magnus_midpoint_step` (problems.py:374-382): host exponential of the
  midpoint generator, device step.

The host helpers (grids, initial states) follow problems.py:273-292,
496-525.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _device as dv
from . import _native
from .errors import ConfigurationError, ShapeError
from .fd import gpe_weighted_factors, sinh_clustered_grid
from .hermite import position_operator
from .kron import KroneckerOp, _cache_mats, prepare, step
from .errors import InvalidReferenceError
from .tensor import _Operand, device_norm, inner_weight_product, norm, run_tucker

__all__ = [
    "VortexProfile",
    "gpe_setup",
    "gpe_strang_run",
    "gpe_strang_step",
    "hkmp_factors",
    "magnus_midpoint_step",
    "relative_error",
    "schrodinger_initial_state",
    "sin2_integral",
    "tdpot_phase_factor",
    "tdpot_strang_step",
    "ti_potentials",
    "vortex_pair_state",
]


# ---------------------------------------------------------------------------
# pointwise operators handed to the C ABI


_inner_weight_product = inner_weight_product


def _gpe_op(shape, weights_dev, half_tau, inner_dev=None, repeat=1):
    op = _native.PointOp()
    op.repeat = repeat
    op.kind = _native.OP_GPE_PHASE
    op.d = len(shape)
    for i, n in enumerate(shape):
        op.dims[i] = n
        op.weights[i] = weights_dev[i].data_ptr()
    op.coef = 0.5 * half_tau  # the i*0.5*half_tau of problems.py:545
    if inner_dev is not None:
        op.inner_weights = inner_dev.data_ptr()
    return op


def _diag_op(shape, factor_dev, direction):
    op = _native.PointOp()
    op.kind = _native.OP_DIAG
    op.d = len(shape)
    for i, n in enumerate(shape):
        op.dims[i] = n
    op.diag = factor_dev.data_ptr()
    op.diag_dir = direction
    return op


def _attach_norm(op, norm_out, dev, keep):
    """Ask the product that applies ``op`` for the two-norm of what it stores (its epilogue's
    per-warp partial sums, folded into ``norm_out[0]``); the partial-sum workspace is
    sized for any product shape (km_norm_epilogue_slots of the largest) and kept alive."""
    dims = [op.dims[i] for i in range(op.d)]
    n = 1
    for x in dims:
        n *= x
    # whichever direction's product ends up applying the op: (rows, fibers) = (n_mu, n / n_mu)
    slots = max(_native.lib().km_norm_epilogue_slots(x, n // x) for x in dims)
    ws = dv.torch.empty(int(slots), dtype=dv.torch.float64, device=dev)
    keep.append(ws)
    op.norm_result = norm_out.data_ptr()
    op.norm_ws = ws.data_ptr()
    op.norm_ws_count = int(slots)


def _check_weights(weights, shape):
    # problems.py:528-539 messages
    if len(weights) != len(shape):
        raise ShapeError(f"expected {len(shape)} weight vectors, got {len(weights)}")
    for ax, w in enumerate(weights):
        wshape = tuple(w.shape) if dv.is_tensor(w) else np.shape(np.asarray(w, dtype=float))
        if wshape != (shape[ax],):
            raise ShapeError(
                f"direction {ax + 1}: weight vector of shape {wshape} does not match extent {shape[ax]}"
            )


def _strang_dtype(psi_dtype, cache):
    # the reference's phase multiplies by a complex128 factor (problems.py:545),
    # so the state leaves the nonlinear half step as complex128 whatever came in
    return np.result_type(psi_dtype, np.complex128, *cache.exp_dtypes())


def _opening_phase_widened(state, op, dev):
    """The opening half-phase of a complex64 state, stored as complex128 (km_pointwise_cast).

    The reference forms the density of a complex64 state in float32
    (``psi.real**2 + psi.imag**2`` on float32 arrays, problems.py:543) and the
    complex128 phase factor promotes the product to complex128 (problems.py:545);
    converting to complex128 first would form the density in float64 instead.
    Returns a column-major complex128 device tensor.
    """
    t = state if dv.is_tensor(state) and state.is_cuda else dv.to_device(np.asarray(state), np.complex64, dev)
    t = dv.tensor_as(t, np.complex64)
    out = dv.fortran_empty(tuple(t.shape), dv.torch.complex128, dev)
    _native.check(_native.lib().km_pointwise_cast(t.data_ptr(), _native.KM_C64, out.data_ptr(), _native.KM_C128,
                                                  t.numel(), ctypes.byref(op), dv.stream_ptr(dev)))
    return out


def gpe_strang_step(linear_cache, weights, psi, tau, _timer=None):
    """One Strang step in the weighted variables (problems.py:548-565).

    ``psi <- N(tau/2) ∘ exp(tau*M) ∘ N(tau/2) psi`` with the exact pointwise
    flow ``N(h) psi = psi * exp(0.5i*h*(1 - |psi|^2/w))``.  ``_timer`` is
    accepted for signature compatibility; device work is asynchronous, so the
    whole step is attributed to it.
    """
    po = _Operand(psi)
    if po.shape != linear_cache.shape:
        raise ShapeError(f"state shape {po.shape} does not match cache shape {linear_cache.shape}")
    _check_weights(weights, po.shape)
    if len(po.shape) > _native.MAX_D:
        raise ConfigurationError(f"the fused Strang step supports at most {_native.MAX_D} directions")
    out_dtype = _strang_dtype(po.dtype, linear_cache)
    dev = po.obj.device if po.is_tensor and po.obj.is_cuda else dv.device()
    w_dev = [dv.cached_vector(w, np.float64, dev) for w in weights]
    inner_dev = dv.cached_vector(_inner_weight_product(weights, po.shape), np.float64, dev) if len(po.shape) > 1 else None
    if inner_dev is not None:
        w_dev.append(inner_dev)  # kept alive with the others
    half_tau = 0.5 * tau
    pre = _gpe_op(po.shape, w_dev, half_tau, inner_dev)
    post = _gpe_op(po.shape, w_dev, half_tau, inner_dev)
    state = po.obj
    host_in = not (po.is_tensor and po.obj.is_cuda)
    if po.dtype == np.complex64 and out_dtype == np.complex128:
        # float32 density in the opening phase, then the complex128 step (see _opening_phase_widened)
        state = _opening_phase_widened(state, pre, dev)
        pre = None
    elif po.dtype != out_dtype and not po.is_tensor:
        state = np.asarray(state).astype(out_dtype, order="F")
    elif po.is_tensor and dv.np_dtype(state.dtype) != out_dtype:
        state = dv.tensor_as(state, out_dtype)
    mats = _cache_mats(linear_cache, _Operand(state))

    def run():
        res = run_tucker(state, mats, pre=pre, post=post, out_dtype=out_dtype, keepalive=w_dev)
        if host_in and dv.is_tensor(res) and not (po.is_tensor and not po.obj.is_cuda):
            return dv.to_host(res)
        if host_in and dv.is_tensor(res):  # CPU torch tensor in -> CPU torch tensor out
            return dv.torch.from_numpy(dv.to_host(res))
        return res

    if _timer is not None:
        with _timer.mode_products():
            return run()
    return run()


def gpe_strang_run(linear_cache, weights, psi, tau, steps, _norm_out=None):
    """``steps`` consecutive :func:`gpe_strang_step` calls (the loop of problems.py:597-598).

    Between two steps the closing half-phase of step k and the opening
    half-phase of step k+1 run back to back inside the fused epilogue of the
    last product (``repeat = 2``), so only the very first half-phase is a
    standalone pass.  Each rotation recomputes the density from the rotated
    value, so the result is bitwise that of the step-by-step loop.
    
    ``_norm_out`` (a one-element float64 device tensor, internal): the two-norm of the
    final state, accumulated in the last product's epilogue (km_pointop.norm_result) -
    the GPE driver's drift (problems.py:596-599) without another pass over the state.
    """
    po = _Operand(psi)
    if po.shape != linear_cache.shape:
        raise ShapeError(f"state shape {po.shape} does not match cache shape {linear_cache.shape}")
    _check_weights(weights, po.shape)
    if steps < 1:
        raise ConfigurationError("need at least one step")
    if len(po.shape) > _native.MAX_D or len(po.shape) < 2:
        raise ConfigurationError(f"the fused Strang run supports 2..{_native.MAX_D} directions")
    out_dtype = _strang_dtype(po.dtype, linear_cache)
    dev = po.obj.device if po.is_tensor and po.obj.is_cuda else dv.device()
    w_dev = [dv.cached_vector(w, np.float64, dev) for w in weights]
    inner_dev = dv.cached_vector(_inner_weight_product(weights, po.shape), np.float64, dev)
    keep = w_dev + [inner_dev]
    half_tau = 0.5 * tau
    single = _gpe_op(po.shape, w_dev, half_tau, inner_dev, 1)
    double = _gpe_op(po.shape, w_dev, half_tau, inner_dev, 2)
    opened = False
    if po.dtype == np.complex64 and out_dtype == np.complex128:
        state = _opening_phase_widened(po.obj, single, dev)  # float32 density, as the reference
        opened = True
    else:
        state = po.obj if po.is_tensor and po.obj.is_cuda else dv.to_device(np.asarray(po.obj), out_dtype, dev)
        state = dv.tensor_as(state, out_dtype)
    mats = _cache_mats(linear_cache, _Operand(state))
    last = single
    if _norm_out is not None:
        last = _gpe_op(po.shape, w_dev, half_tau, inner_dev, 1)
        _attach_norm(last, _norm_out, dev, keep)
    for k in range(steps):
        pre = single if (k == 0 and not opened) else None
        post = last if k == steps - 1 else double
        state = run_tucker(state, mats, pre=pre, post=post, out_dtype=out_dtype, keepalive=keep)
    if po.is_tensor and po.obj.is_cuda:
        return state
    return dv.to_host(state)


def relative_error(u, ref, norm_kind="max", weights=None):
    """``|u - ref| / |ref|`` in the chosen norm (problems.py:160-169), on the device.

    The difference is formed inside the reduction kernel (no temporary tensor).
    """
    uo, ro = _Operand(u), _Operand(ref)
    if uo.shape != ro.shape:
        raise ShapeError(f"shapes {uo.shape} and {ro.shape} differ")
    denom = norm(ref, norm_kind, weights)
    if denom == 0.0:
        raise InvalidReferenceError("reference tensor has zero norm")
    return device_norm(uo.obj, norm_kind, weights, b=ro.obj) / denom


def sin2_integral(t_a, t_b):
    """``∫_{t_a}^{t_b} sin(s)^2 ds = [s/2 - sin(2s)/4]``."""
    return (t_b / 2 - math.sin(2 * t_b) / 4) - (t_a / 2 - math.sin(2 * t_a) / 4)


def tdpot_phase_factor(x, t_a, t_b):
    """Exact flow of ``i psi' = x sin(t)^2 psi`` over [t_a, t_b]: ``exp(-i x ∫ sin^2)``."""
    return np.exp(-1j * np.asarray(x, dtype=float) * sin2_integral(t_a, t_b))


def tdpot_strang_step(linear_cache, x_nodes, psi, t, tau, direction=3):
    """One Strang step of ``i psi' = (H_0 + x_dir sin(t)^2) psi`` (configuration 4).

    ``linear_cache`` holds the exact propagators of ``H_0`` for ``tau``
    (e.g. :func:`hermite.physical_propagator` per direction); the potential
    flow ``exp(-i x ∫ sin^2)`` over [t, t+tau/2] is applied before and over
    [t+tau/2, t+tau] after it.  Both flows are diagonal along ``direction``
    and the products along the other directions commute with them, so they
    are folded into that direction's propagator on the device,
    ``diag(f_b) E diag(f_a)`` (``km_diag_phase_fold``: the phases are formed
    from the node vector and two scalars, nothing is uploaded per step), and
    the step is a plain d-product Tucker launch: no pointwise pass at all.  Against applying the two phases separately the results differ
    only in rounding (tests/test_gpu_parity.py).
    """
    po = _Operand(psi)
    if po.shape != linear_cache.shape:
        raise ShapeError(f"state shape {po.shape} does not match cache shape {linear_cache.shape}")
    if not 1 <= direction <= len(po.shape):
        raise ShapeError(f"potential direction {direction} outside 1..{len(po.shape)}")
    x = np.asarray(x_nodes, dtype=float)
    if x.shape != (po.shape[direction - 1],):
        raise ShapeError(f"direction {direction}: node vector of shape {x.shape} does not match extent "
                         f"{po.shape[direction - 1]}")
    out_dtype = _strang_dtype(po.dtype, linear_cache)
    dev = po.obj.device if po.is_tensor and po.obj.is_cuda else dv.device()
    c_a, c_b = sin2_integral(t, t + 0.5 * tau), sin2_integral(t + 0.5 * tau, t + tau)
    state = po.obj
    if po.dtype != out_dtype and not po.is_tensor:
        state = np.asarray(state).astype(out_dtype, order="F")
    elif po.is_tensor and dv.np_dtype(state.dtype) != out_dtype:
        state = dv.tensor_as(state, out_dtype)
    mats = _cache_mats(linear_cache, _Operand(state))
    k = direction - 1
    e = mats[k] if mats[k].dtype == dv.torch.complex128 else mats[k].to(dv.torch.complex128)
    x_dev = dv.cached_vector(x, np.float64, dev)
    folded = dv.torch.empty_like(e)
    _native.check(_native.lib().km_diag_phase_fold(e.data_ptr(), folded.data_ptr(), e.shape[0], e.shape[1],
                                                   x_dev.data_ptr(), x_dev.data_ptr(), c_a, c_b,
                                                   dv.stream_ptr(dev)))
    mats[k] = folded
    return run_tucker(state, mats, out_dtype=out_dtype, keepalive=(x_dev, e))


def magnus_midpoint_step(factors_of_t, u, t, tau, device_expm=False):
    """Exponential midpoint rule ``u <- exp(tau * M(t + tau/2)) u`` (problems.py:374-382).

    By default the midpoint exponentials are host scipy ``expm``, as in the
    reference; the step is the device Tucker product, and host work for the
    next call overlaps the device work of this one because device launches
    are asynchronous.  ``device_expm=True`` takes the exponentials on the GPU
    as well (:mod:`expm`).
    """
    op = factors_of_t(t + 0.5 * tau)
    if device_expm:
        from .expm import prepare_device

        return step(prepare_device(op, tau), u)
    return step(prepare(op, tau), u)


def hkmp_factors(basis, t):
    """Coefficient-space generator of the driven oscillator at time t (problems.py:385-394)."""
    d_harm = np.diag(np.arange(basis.k) + 0.5)
    a_static = -1j * d_harm
    a_driven = -1j * (d_harm + np.sin(t) ** 2 * position_operator(basis))
    return KroneckerOp((a_static, a_static, a_driven))


# ---------------------------------------------------------------------------
# host setup (problems.py:273-292, 496-525)


def schrodinger_initial_state(axes):
    """``2^(-5/2) π^(-3/4) (x1 + i x2) exp(-(x1²+x2²+x3²)/4)`` on a tensor grid."""
    x1 = np.asarray(axes[0], dtype=float)[:, None, None]
    x2 = np.asarray(axes[1], dtype=float)[None, :, None]
    x3 = np.asarray(axes[2], dtype=float)[None, None, :]
    env = np.exp(-(x1**2) / 4) * np.exp(-(x2**2) / 4) * np.exp(-(x3**2) / 4)
    return np.asfortranarray(2.0**-2.5 * np.pi**-0.75 * (x1 + 1j * x2) * env)


def ti_potentials():
    """Per-direction potentials of the time-independent benchmark (problems.py:286-292)."""
    return (lambda x: np.cos(2 * np.pi * x), lambda x: 0.5 * x * x, lambda x: 0.5 * x * x)


@dataclass(frozen=True)
class VortexProfile:
    """Rational core profile ``f(r)`` of a straight vortex line (problems.py:477-493)."""

    a1: float = 11.0 / 32.0
    a2: float = 11.0 / 384.0
    b1: float = 1.0 / 3.0
    offset: float = 2.0

    def radial(self, r):
        r2 = np.asarray(r) ** 2
        return np.sqrt(r2 * (self.a1 + self.a2 * r2) / (1.0 + self.b1 * r2 + self.a2 * r2**2))


def vortex_pair_state(grids, profile=VortexProfile()):
    """Two orthogonal straight vortices in a unit background (problems.py:496-512)."""
    x1 = grids[0].points[:, None, None]
    x2 = grids[1].points[None, :, None]
    x3 = grids[2].points[None, None, :]
    dlt = profile.offset
    psi_a = profile.radial(np.sqrt(x2**2 + (x3 + dlt) ** 2)) * np.exp(1j * np.arctan2(x3 + dlt, x2))
    psi_b = profile.radial(np.sqrt((x3 - dlt) ** 2 + x1**2)) * np.exp(1j * np.arctan2(x1, x3 - dlt))
    return np.asfortranarray(psi_a * psi_b)


def gpe_setup(n, half_width=20.0, strength=2.0):
    """Clustered grids, ``i *`` symmetrised half-Laplacian factors, trapezoid weights (problems.py:515-525)."""
    grids = tuple(sinh_clustered_grid(n, half_width, strength) for _ in range(3))
    sym_op, weights = gpe_weighted_factors(grids)
    return grids, KroneckerOp(tuple(1j * a for a in sym_op.factors)), weights


def weighted_vortex_state(grids, weights):
    """``sqrt(w_1 w_2 w_3) * vortex_pair_state`` in F order (problems.py:589-592)."""
    psi = vortex_pair_state(grids)
    for ax, w in enumerate(weights):
        psi = psi * np.sqrt(w).reshape((1,) * ax + (w.size,) + (1,) * (2 - ax))
    return np.asfortranarray(psi)

