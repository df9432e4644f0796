"""Dense order-d tensor kernels on the B200: μ-mode products, Tucker operator, norms.

Drop-in for the reference's ``kronmode.tensor`` (tensor.py:1-199).  Tensors
are column-major (direction 1 fastest, tensor.py:3-6); directions are
1-based.  Every product runs on the GPU through ``libkmb200.so``
(include/kmb200.h ``km_mumode`` / ``km_tucker``) — one DMMA GEMM per product
over the (n_left, n_mu, n_right) flattening of tensor.py:132-134.

Inputs may be numpy arrays (copied to the device and back: numpy in → numpy
out, F-ordered, as the reference returns) or CUDA torch tensors with
column-major strides (kept on the device: tensor in → tensor out).
Validation, error classes and messages, dtype promotion (``np.result_type``,
tensor.py:113) and the multiply-add tally (tensor.py:114-115) follow the
reference so its tests read the same.
"""

from __future__ import annotations

import ctypes
from contextlib import contextmanager
from math import prod

import numpy as np

from . import _device as dv
from . import _native
from . import _pipeline
from .errors import ConfigurationError, InvalidDirectionError, ShapeError

__all__ = [
    "FlopCounter",
    "count_flops",
    "mu_fiber_count",
    "mu_mode_product",
    "norm",
    "tucker",
]


class FlopCounter:
    """Multiply-add tally of the mode products executed while armed (tensor.py:34-40)."""

    __slots__ = ("macs",)

    def __init__(self):
        self.macs = 0


_active_counters: list[FlopCounter] = []


@contextmanager
def count_flops():
    """Arm a :class:`FlopCounter` for mode products run inside the block (tensor.py:46-59).

    One ``m x n_mu`` product applied to a tensor with ``N/n_mu`` fibers adds
    ``m * (N/n_mu) * n_mu`` multiply-adds.
    """
    counter = FlopCounter()
    _active_counters.append(counter)
    try:
        yield counter
    finally:
        _active_counters.remove(counter)


def _tally(macs):
    for counter in _active_counters:
        counter.macs += macs


def _check_direction(ndim, mu):
    # tensor.py:62-66
    if not isinstance(mu, (int, np.integer)) or isinstance(mu, bool):
        raise InvalidDirectionError(f"direction index must be an integer, got {mu!r}")
    if not 1 <= mu <= ndim:
        raise InvalidDirectionError(f"direction {mu} outside 1..{ndim}")


def mu_fiber_count(shape, mu):
    """Number of mu-fibers of a tensor with the given extents, ``N / n_mu`` (tensor.py:69-77)."""
    dims = tuple(int(n) for n in shape)
    if not dims:
        raise ShapeError("shape must have at least one extent")
    if any(n < 1 for n in dims):
        raise ShapeError(f"extents must be positive, got {dims}")
    _check_direction(len(dims), mu)
    return prod(dims) // dims[mu - 1]


# --------------------------------------------------------------------------
# operand handling


class _Operand:
    """A tensor or matrix argument: numpy/torch, its shape and numpy dtype."""

    __slots__ = ("obj", "shape", "dtype", "is_tensor")

    def __init__(self, obj):
        self.is_tensor = dv.is_tensor(obj)
        if self.is_tensor:
            self.obj = obj
            self.shape = tuple(obj.shape)
            self.dtype = dv.np_dtype(obj.dtype)
        else:
            self.obj = np.asarray(obj)
            self.shape = self.obj.shape
            self.dtype = self.obj.dtype

    @property
    def ndim(self):
        return len(self.shape)


def _compute_dtype(out_dtype):
    """Device dtype for a numpy result dtype (f16/ints/bools are widened)."""
    out_dtype = np.dtype(out_dtype)
    if out_dtype in dv.SUPPORTED:
        return out_dtype
    if out_dtype.kind == "c":
        return np.dtype(np.complex128)
    if out_dtype == np.float16:
        return np.dtype(np.float32)
    if out_dtype.kind in "biuf":
        return np.dtype(np.float64)
    raise ConfigurationError(f"unsupported dtype {out_dtype} for a mode product")


def _operand_dtype(dtype, single):
    cplx = np.dtype(dtype).kind == "c"
    if single:
        return np.dtype(np.complex64 if cplx else np.float32)
    return np.dtype(np.complex128 if cplx else np.float64)


def _tensor_on_device(op, dtype, dev):
    if op.is_tensor:
        t = op.obj
        if t.device != dev:
            t = t.to(dev)
        return dv.tensor_as(t, dtype)
    return dv.to_device(op.obj, dtype, dev)


_TC_WORKSPACE = {}
_RR32_ON_TC = True  # float32 x float32 fiber pairs on tcgen05 (False: DMMA; for A/B probes)
# below this many elements the DMMA route wins (tools/f32_probe.py: 128^3 90 against 130 us,
# 256^3 1174 against 468 us per step)
_RR32_MIN_ELEMENTS = 1 << 23


def launch_product(src_ptr, src_code, mat_ptr, mat_code, dst_ptr, m, nl, nmu, nr, op, stream, dev):
    """One μ-mode product through the C ABI: complex64 x complex64 on the tcgen05
    (TF32x3) kernel, everything else on the DMMA kernels."""
    lib = _native.lib()
    if src_code == _native.KM_C64 and mat_code == _native.KM_C64 and op is None:
        need = ctypes.c_size_t(0)
        _native.check(lib.km_tc_workspace_bytes(m, nmu, ctypes.byref(need)))
        # one workspace per (device, stream): calls on one stream are ordered, so
        # the factor planes of consecutive products may share it
        key = (str(dev), stream.value if isinstance(stream, ctypes.c_void_p) else stream)
        buf = _TC_WORKSPACE.get(key)
        if buf is None or buf.numel() < need.value:
            buf = dv.torch.empty(need.value, dtype=dv.torch.uint8, device=dev)
            _TC_WORKSPACE[key] = buf
        _native.check(lib.km_mumode_c64_tc(src_ptr, mat_ptr, dst_ptr, m, nl, nmu, nr, buf.data_ptr(),
                                           buf.numel(), stream))
        return
    _native.check(lib.km_mumode(src_ptr, src_code, mat_ptr, mat_code, dst_ptr, m, nl, nmu, nr,
                                None if op is None else ctypes.byref(op), stream))


def run_tucker(u, mats, pre=None, post=None, out_dtype=None, keepalive=()):
    """:func:`_run_tucker` with the tensor's device current (the C ABI launches on the current
    device: a CUDA tensor on another GPU than the current one is handled there)."""
    uo = u.device if dv.is_tensor(u) and u.is_cuda else None
    with dv.on_device(uo):
        return _run_tucker(u, mats, pre, post, out_dtype, keepalive)


_TORCH_SAME_PRECISION = {}
if dv.torch is not None:
    _t = dv.torch
    for _u in (_t.float64, _t.complex128):
        for _m in (_t.float64, _t.complex128):
            _TORCH_SAME_PRECISION[(_u, _m)] = _m
    for _u in (_t.float32, _t.complex64):
        for _m in (_t.float32, _t.complex64):
            _TORCH_SAME_PRECISION[(_u, _m)] = _m

_PLANS = {}
_PLANS_MAX = 256


def _fast_tucker(u, mats, pre, post, out_dtype, keepalive):
    """The device-resident case of :func:`_run_tucker` from a per-shape plan.

    A column-major CUDA tensor with device-tensor factors of its own precision (e.g. a
    PropagatorCache's device copies) needs none of the dtype walks, workspace queries and
    ctypes array builds per call: they are memoised per (shapes, dtypes, op presence,
    device).  Returns None when the plan does not apply (the general path then runs).
    """
    if not dv.is_fortran(u) or len(mats) > _native.MAX_D or \
            not all(m is None or dv.is_tensor(m) for m in mats):
        return None
    key = (tuple(u.shape), u.dtype, u.device, out_dtype,
           tuple(None if m is None else (tuple(m.shape), m.dtype, m.device, m.is_contiguous()) for m in mats),
           pre is None, post is None, None if pre is None else pre.kind, None if post is None else post.kind)
    plan = _PLANS.get(key)
    if plan is None:
        if any(m is not None and (not dv.is_tensor(m) or m.device != u.device or not m.is_contiguous()
                                  or m.dtype != _TORCH_SAME_PRECISION.get((u.dtype, m.dtype), None))
               for m in mats):
            _PLANS[key] = False
            return None
        plan = _make_plan(u, mats, pre, post, out_dtype)
        if len(_PLANS) >= _PLANS_MAX:
            _PLANS.pop(next(iter(_PLANS)))
        _PLANS[key] = plan
    if plan is False:
        return None
    (d, out_shape, cdt_t, u_code, c_dims, c_codes, c_rows, need, fits, nact, macs, finish_dt) = plan
    for mac in macs:
        _tally(mac)
    dev = u.device
    lib = _native.lib()
    out = dv.fortran_empty(out_shape, cdt_t, dev)
    c_mats = (ctypes.c_void_p * d)(*[None if m is None else m.data_ptr() for m in mats])
    ws0 = dv.torch.empty(max(need, 1), dtype=dv.torch.uint8, device=dev) if need else None
    ws1 = dv.torch.empty(max(need, 1), dtype=dv.torch.uint8, device=dev) if need and nact > 1 and not fits else None
    _native.check(lib.km_tucker(
        u.data_ptr(), u_code, d, c_dims, c_mats, c_codes, c_rows, out.data_ptr(),
        None if ws0 is None else ws0.data_ptr(), None if ws1 is None else ws1.data_ptr(),
        None if pre is None else ctypes.byref(pre), None if post is None else ctypes.byref(post),
        dv.stream_ptr(dev)))
    del ws0, ws1, keepalive
    if finish_dt is not None:
        out = dv.tensor_as(out, finish_dt)
    return out


class StepPlan:
    """A fully prebuilt ``km_tucker`` call for fixed device factors (a PropagatorCache's):
    ctypes arrays, workspace size, output shape and dtype, and, for small states, one reusable
    scratch buffer per stream (calls on one stream are ordered, so consecutive steps may share
    it).  The hot loop of small states calls ``run`` and nothing else (kron.step's fast path).
    Scratch above ``KEEP_WS_BYTES`` is taken from torch's allocator per call instead, so a cache
    kept alive does not pin a state-sized buffer (and a new cache per step, as in the Magnus
    driver, does not allocate one per step)."""

    KEEP_WS_BYTES = 32 << 20

    __slots__ = ("mats", "plan", "c_mats", "ws", "dev")

    def __init__(self, u, mats):
        self.mats = tuple(mats)
        same = all(m is None or (dv.is_tensor(m) and m.device == u.device and m.is_contiguous()
                                 and m.dtype == _TORCH_SAME_PRECISION.get((u.dtype, m.dtype)))
                   for m in self.mats)
        self.plan = _make_plan(u, self.mats, None, None, None) if same else False
        self.dev = u.device
        if self.plan is not False:
            d = self.plan[0]
            self.c_mats = (ctypes.c_void_p * d)(*[None if m is None else m.data_ptr() for m in self.mats])
        self.ws = {}

    @property
    def ok(self):
        return self.plan is not False

    def run(self, u):
        (d, out_shape, cdt_t, u_code, c_dims, c_codes, c_rows, need, fits, nact, macs, finish_dt) = self.plan
        for mac in macs:
            _tally(mac)
        dev = self.dev
        stream = dv.stream_ptr(dev)
        out = dv.fortran_empty(out_shape, cdt_t, dev)
        ws0 = ws1 = None
        if need > self.KEEP_WS_BYTES:
            ws0 = dv.torch.empty(need, dtype=dv.torch.uint8, device=dev)
            if nact > 1 and not fits:
                ws1 = dv.torch.empty(need, dtype=dv.torch.uint8, device=dev)
        elif need:
            bufs = self.ws.get(stream.value)
            if bufs is None:
                n1 = 2 if (nact > 1 and not fits) else 1
                bufs = [dv.torch.empty(max(need, 1), dtype=dv.torch.uint8, device=dev) for _ in range(n1)]
                if len(self.ws) >= 4:
                    self.ws.pop(next(iter(self.ws)))
                self.ws[stream.value] = bufs
            ws0 = bufs[0]
            ws1 = bufs[1] if len(bufs) > 1 else None
        _native.check(_native.lib().km_tucker(
            u.data_ptr(), u_code, d, c_dims, self.c_mats, c_codes, c_rows, out.data_ptr(),
            None if ws0 is None else ws0.data_ptr(), None if ws1 is None else ws1.data_ptr(), None, None, stream))
        if finish_dt is not None:
            out = dv.tensor_as(out, finish_dt)
        return out


def _make_plan(u, mats, pre, post, out_dtype):
    d = u.dim()
    udt = dv.np_dtype(u.dtype)
    result = np.result_type(udt, *[dv.np_dtype(m.dtype) for m in mats if m is not None])
    if out_dtype is not None:
        result = np.result_type(result, out_dtype)
    cdt = _compute_dtype(result)
    phased = any(op is not None and op.kind != _native.OP_NONE for op in (pre, post))
    if phased and udt.kind != "c":
        return False
    if udt == np.dtype(np.complex64) and any(m is not None and not m.is_complex() for m in mats):
        return False  # complex64 x real float32: the general path promotes the factor (tcgen05)
    cur, macs, codes, rows = list(u.shape), [], [], []
    for mu, m in enumerate(mats):
        if m is None:
            codes.append(0)
            rows.append(0)
            continue
        macs.append(m.shape[0] * prod(cur))
        cur[mu] = m.shape[0]
        codes.append(dv.code(dv.np_dtype(m.dtype)))
        rows.append(m.shape[0])
    out_shape = tuple(cur)
    if any(n == 0 for n in u.shape) or any(n == 0 for n in out_shape):
        return False
    for tdt, tcode in ((np.dtype(np.complex64), _native.KM_C64), (np.dtype(np.float32), _native.KM_F32)):
        if udt == tdt and pre is None and post is None and \
                all(c == tcode for m, c in zip(mats, codes) if m is not None):
            return False  # the tcgen05 loop (per-product launches) of the general path
    c_dims = (ctypes.c_int64 * d)(*u.shape)
    c_codes = (ctypes.c_int * d)(*codes)
    c_rows = (ctypes.c_int64 * d)(*rows)
    c_probe = (ctypes.c_void_p * d)(*[None if m is None else 1 for m in mats])
    ws = ctypes.c_size_t(0)
    u_code = dv.code(udt)
    _native.check(_native.lib().km_tucker_workspace(u_code, d, c_dims, c_probe, c_codes, c_rows, ctypes.byref(ws)))
    nact = sum(m is not None for m in mats)
    need = ws.value if (nact > 1 or pre is not None) else 0
    out_bytes = prod(out_shape) * cdt.itemsize
    fits = need <= out_bytes
    finish_dt = result if result != cdt and result in dv.SUPPORTED else None
    if result != cdt and result not in dv.SUPPORTED:
        return False
    return (d, out_shape, dv.torch_dtype(cdt), u_code, c_dims, c_codes, c_rows, need, fits, nact, macs, finish_dt)


def _run_tucker(u, mats, pre=None, post=None, out_dtype=None, keepalive=()):
    """Core device driver: ``post(pre(u) x_1 mats[0] ... x_d mats[d-1])``.

    ``u``/``mats`` are already validated.  ``pre``/``post`` are
    :class:`_native.PointOp` (or None).  ``out_dtype`` forces a result dtype
    (used by the splitting schemes).  Returns numpy for numpy input and a
    device tensor for tensor input.
    """
    if dv.is_tensor(u) and u.is_cuda:
        res = _fast_tucker(u, mats, pre, post, out_dtype, keepalive)
        if res is not None:
            return res
    uo = _Operand(u)
    mos = [None if m is None else _Operand(m) for m in mats]
    d = uo.ndim
    result = np.result_type(uo.dtype, *[m.dtype for m in mos if m is not None])
    if out_dtype is not None:
        result = np.result_type(result, out_dtype)
    cdt = _compute_dtype(result)
    single = cdt in (np.dtype(np.float32), np.dtype(np.complex64))
    u_dt = _operand_dtype(uo.dtype, single)
    # a phase op needs a complex state (a post carrying only the epilogue norm does not)
    phased = any(op is not None and op.kind != _native.OP_NONE for op in (pre, post))
    if phased and u_dt.kind != "c":
        u_dt = _operand_dtype(np.complex64, single)

    # the reference's per-product multiply-add tally (tensor.py:114-115)
    cur = list(uo.shape)
    for mu, m in enumerate(mos):
        if m is None:
            continue
        _tally(m.shape[0] * prod(cur))
        cur[mu] = m.shape[0]
    out_shape = tuple(cur)

    dev = uo.obj.device if uo.is_tensor and uo.obj.is_cuda else dv.device()
    if any(n == 0 for n in uo.shape) or any(n == 0 for n in out_shape):
        return _finish(uo, dv.fortran_empty(out_shape, dv.torch_dtype(cdt), dev).zero_(), result, cdt)

    mats_dev, codes, rows = [], [], []
    for m in mos:
        if m is None:
            mats_dev.append(None)
            codes.append(0)
            rows.append(0)
            continue
        mdt = _operand_dtype(m.dtype, single)
        if single and u_dt.kind == "c" and mdt.kind != "c":
            # single precision, complex state, real factor (e.g. the float32 Hermite basis):
            # the reference's np.matmul promotes the factor to complex64 (zero imaginary
            # parts) and computes in complex64; so do we, on the tcgen05 kernel (3xTF32)
            # instead of the FP64 DMMA kernel (about 3.5x faster even with the zeros)
            mdt = np.dtype(np.complex64)
        mats_dev.append(dv.cached_vector(m.obj, mdt, dev))
        codes.append(dv.code(mdt))
        rows.append(m.shape[0])

    if not uo.is_tensor and _pipeline.eligible(uo.obj, d):
        # host in / host out: overlap the PCIe copies with the products
        host = np.asfortranarray(uo.obj if uo.dtype == u_dt else uo.obj.astype(u_dt, order="F"))
        res = _pipeline.tucker_host_pipelined(host, u_dt, mats_dev, codes, rows, pre, post, out_shape, cdt, dev)
        del keepalive
        return res if res.dtype == result else res.astype(result, order="F")

    u_dev = _tensor_on_device(uo, u_dt, dev)
    lib = _native.lib()
    out = dv.fortran_empty(out_shape, dv.torch_dtype(cdt), dev)
    stream = dv.stream_ptr(dev)
    c64 = np.dtype(np.complex64)
    tc_loop = (u_dt == c64 and pre is None and post is None
               and all(c == _native.KM_C64 for t, c in zip(mats_dev, codes) if t is not None))
    # float32 x float32 on large states: products whose fibers come in pairs (n_left even) run on
    # the tcgen05 kernel too, two real fibers read as one complex64 fiber (E z = E u_f + i E u_f+1,
    # exact) against the factor widened to complex64; direction 1 (n_left = 1) stays on DMMA
    rr32 = (_RR32_ON_TC and u_dt == np.dtype(np.float32) and pre is None and post is None
            and prod(uo.shape) >= _RR32_MIN_ELEMENTS
            and all(c == _native.KM_F32 for t, c in zip(mats_dev, codes) if t is not None))
    tc_loop = tc_loop or rr32
    if d <= _native.MAX_D and not tc_loop:
        c_dims = (ctypes.c_int64 * d)(*uo.shape)
        c_mats = (ctypes.c_void_p * d)(*[None if t is None else t.data_ptr() for t in mats_dev])
        c_codes = (ctypes.c_int * d)(*codes)
        c_rows = (ctypes.c_int64 * d)(*rows)
        ws = ctypes.c_size_t(0)
        u_code = dv.code(u_dt)
        _native.check(lib.km_tucker_workspace(u_code, d, c_dims, c_mats, c_codes, c_rows, ctypes.byref(ws)))
        nact = sum(t is not None for t in mats_dev)
        need = ws.value if (nact > 1 or pre is not None) else 0
        ws0 = dv.torch.empty(max(need, 1), dtype=dv.torch.uint8, device=dev) if need else None
        # out doubles as the second ping-pong buffer when every intermediate fits in it
        fits = need <= out.numel() * out.element_size()
        ws1 = dv.torch.empty(max(need, 1), dtype=dv.torch.uint8, device=dev) if need and nact > 1 and not fits else None
        _native.check(
            lib.km_tucker(
                u_dev.data_ptr(), u_code, d, c_dims, c_mats, c_codes, c_rows, out.data_ptr(),
                None if ws0 is None else ws0.data_ptr(), None if ws1 is None else ws1.data_ptr(),
                None if pre is None else ctypes.byref(pre), None if post is None else ctypes.byref(post),
                stream,
            )
        )
        del ws0, ws1, keepalive
    else:
        if pre is not None or post is not None:
            raise ConfigurationError(f"pointwise phases support at most {_native.MAX_D} directions")
        src, src_dt, shape = u_dev, u_dt, list(uo.shape)
        active = [mu for mu, t in enumerate(mats_dev) if t is not None]
        if not active:
            out.copy_(src)
        for idx, mu in enumerate(active):
            mdt = _operand_dtype(mos[mu].dtype, single)
            new_dt = np.result_type(src_dt, mdt)
            shape_new = list(shape)
            shape_new[mu] = rows[mu]
            dst = out if idx == len(active) - 1 else dv.fortran_empty(shape_new, dv.torch_dtype(new_dt), dev)
            nl = prod(shape[:mu])
            if rr32 and nl % 2 == 0:
                launch_product(src.data_ptr(), _native.KM_C64, dv.cached_vector(mos[mu].obj, c64, dev).data_ptr(),
                               _native.KM_C64, dst.data_ptr(), rows[mu], nl // 2, shape[mu], prod(shape[mu + 1:]),
                               None, stream, dev)
            else:
                launch_product(src.data_ptr(), dv.code(src_dt), mats_dev[mu].data_ptr(), codes[mu], dst.data_ptr(),
                               rows[mu], nl, shape[mu], prod(shape[mu + 1:]), None, stream, dev)
            src, src_dt, shape = dst, new_dt, shape_new
    return _finish(uo, out, result, cdt)


def kronecker_sum_apply(t, mats, out=None):
    """``sum_mu t x_mu mats[mu]`` on the device in d launches (kron.py:94-102).

    ``t`` is a column-major CUDA tensor and ``mats`` square device matrices, all
    of one precision; the first product writes ``out`` (column-major, the
    promoted dtype), every later one accumulates into it in its epilogue
    (km_mumode_split accumulate = 1: ``out += p`` rounded as numpy does), so the
    sum costs no extra HBM pass and no temporary.  A real tensor with complex
    factors is widened first (every term must be of the output dtype).
    """
    lib = _native.lib()
    shape = tuple(t.shape)
    dev = t.device
    cdt = np.result_type(dv.np_dtype(t.dtype), *[dv.np_dtype(m.dtype) for m in mats])
    if dv.np_dtype(t.dtype) != cdt:
        t = dv.tensor_as(t, cdt)
    t = dv.as_fortran(t)
    if out is None:
        out = dv.fortran_empty(shape, dv.torch_dtype(cdt), dev)
    stream = dv.stream_ptr(dev)
    code = dv.code(cdt)
    for mu, m in enumerate(mats):
        n = shape[mu]
        nl, nr = prod(shape[:mu]), prod(shape[mu + 1:])
        _tally(n * prod(shape))
        _native.check(lib.km_mumode_split(t.data_ptr(), code, m.data_ptr(), dv.code(dv.np_dtype(m.dtype)),
                                          out.data_ptr(), n, nl, n, nr, n, 0, n, 0, 1 if mu else 0, None, stream))
    return out


def _finish(uo, out, result, cdt):
    if uo.is_tensor and uo.obj.is_cuda:
        if result != cdt:
            out = dv.tensor_as(out, result) if result in dv.SUPPORTED else out.to(dv.torch_dtype(result))
        return out
    host = dv.to_host(out)
    if host.dtype != result:
        host = host.astype(result, order="F")
    if uo.is_tensor:  # CPU torch tensor in → CPU torch tensor out
        return dv.torch.from_numpy(host)
    return host


# --------------------------------------------------------------------------
# public API


def mu_mode_product(u, mat, mu):
    """Multiply ``mat`` onto every mu-fiber of ``u`` (tensor.py:80-140).

    Returns a column-major tensor of shape ``(n_1, ..., m, ..., n_d)`` with
    ``S[..., i, ...] = sum_j mat[i, j] * u[..., j, ...]``; real and complex
    operands mix by numpy promotion.  Computed on the GPU as one DMMA GEMM.
    """
    uo = _Operand(u)
    mo = _Operand(mat)
    _check_direction(uo.ndim, mu)
    if mo.ndim != 2:
        raise ShapeError(f"operator for direction {mu} must be a matrix, got ndim={mo.ndim}")
    n_mu = uo.shape[mu - 1]
    if mo.shape[1] != n_mu:
        raise ShapeError(f"direction {mu}: matrix has {mo.shape[1]} columns, tensor extent is {n_mu}")
    mats = [None] * uo.ndim
    mats[mu - 1] = mo.obj
    return run_tucker(uo.obj, mats)


def _validate_tucker(uo, mats):
    # tensor.py:150-161: every slot is checked before any work
    if len(mats) != uo.ndim:
        raise ShapeError(f"expected {uo.ndim} matrix slots, got {len(mats)}")
    for mu, mat in enumerate(mats, start=1):
        if mat is None:
            continue
        mo = _Operand(mat)
        if mo.ndim != 2 or mo.shape[1] != uo.shape[mu - 1]:
            raise ShapeError(
                f"direction {mu}: matrix of shape {mo.shape} does not act on extent {uo.shape[mu - 1]}"
            )


def tucker(u, mats):
    """Apply one matrix per direction: ``u x_1 mats[0] x_2 ... x_d mats[d-1]`` (tensor.py:143-166).

    ``None`` entries are skipped; directions are applied in ascending order.
    """
    uo = _Operand(u)
    mats = list(mats)
    _validate_tucker(uo, mats)
    if all(m is None for m in mats):
        return u if uo.is_tensor else uo.obj
    return run_tucker(uo.obj, mats)


def inner_weight_product(weights, shape):
    """w_1 ... w_{d-1} accumulated left to right (problems.py:528-539), flattened column-major."""
    d = len(shape)
    inner = np.ones(shape[:-1], order="F")
    for ax, w in enumerate(weights[:-1]):
        w = w.detach().cpu().numpy() if dv.is_tensor(w) else np.asarray(w, dtype=float)
        inner *= w.reshape((1,) * ax + (w.size,) + (1,) * (d - 2 - ax))
    return inner.reshape(-1, order="F")


_NORM_KIND = {"max": 0, "two": 1, "weighted_two": 2}
_NORM_WS = {}


def device_norm(a, kind, weights=None, b=None):
    """||a - b|| (b optional) through the ``km_norm`` kernels; ``a``/``b`` numpy or CUDA tensors."""
    with dv.on_device(a.device if dv.is_tensor(a) and a.is_cuda else None):
        return _device_norm(a, kind, weights, b)


def _device_norm(a, kind, weights=None, b=None):
    ao = _Operand(a)
    dev = ao.obj.device if ao.is_tensor and ao.obj.is_cuda else dv.device()
    dt = _compute_dtype(np.result_type(ao.dtype, *([] if b is None else [_Operand(b).dtype])))
    ta = _tensor_on_device(ao, dt, dev)
    tb = None if b is None else _tensor_on_device(_Operand(b), dt, dev)
    lib = _native.lib()
    key = str(dev)
    ws = _NORM_WS.get(key)
    if ws is None:
        ws = dv.torch.empty(lib.km_norm_workspace_bytes() + 8, dtype=dv.torch.uint8, device=dev)
        _NORM_WS[key] = ws
    result = dv.torch.empty(1, dtype=dv.torch.float64, device=dev)
    op = None
    keep = []
    if kind == "weighted_two":
        shape = ao.shape if len(ao.shape) >= 2 else (1,) + tuple(ao.shape)
        wl = list(weights) if len(ao.shape) >= 2 else [np.ones(1), weights[0]]
        inner = dv.cached_vector(inner_weight_product(wl, shape), np.float64, dev)
        last = dv.cached_vector(wl[-1], np.float64, dev)
        keep = [inner, last]
        op = _native.PointOp()
        op.kind = _native.OP_GPE_PHASE
        op.d = len(shape)
        for i, n in enumerate(shape):
            op.dims[i] = n
        op.weights[len(shape) - 1] = last.data_ptr()
        op.inner_weights = inner.data_ptr()
    _native.check(lib.km_norm(ta.data_ptr(), None if tb is None else tb.data_ptr(), dv.code(dt), ta.numel(),
                              _NORM_KIND[kind], None if op is None else ctypes.byref(op), result.data_ptr(),
                              ws.data_ptr(), ws.numel(), dv.stream_ptr(dev)))
    del keep
    return float(result.item())


def norm(u, kind="two", weights=None):
    """Tensor norm: ``max``, Euclidean ``two`` or ``weighted_two`` (tensor.py:169-198).

    One deterministic device reduction (``km_norm``: fixed grid, fixed order).
    """
    uo = _Operand(u)
    if kind not in ("max", "two", "weighted_two"):
        raise ConfigurationError(f"unknown norm kind {kind!r}")
    if kind == "weighted_two":
        if weights is None:
            raise ConfigurationError("weighted_two norm requires per-direction weights")
        if len(weights) != uo.ndim:
            raise ShapeError(f"expected {uo.ndim} weight vectors, got {len(weights)}")
        for mu, w in enumerate(weights, start=1):
            wshape = tuple(np.shape(w)) if not dv.is_tensor(w) else tuple(w.shape)
            if wshape != (uo.shape[mu - 1],):
                raise ShapeError(
                    f"direction {mu}: weight vector of shape {wshape} does not match "
                    f"extent {uo.shape[mu - 1]}"
                )
    if uo.ndim == 0:
        return float(abs(np.asarray(uo.obj if not uo.is_tensor else uo.obj.cpu()).item()))
    if any(n == 0 for n in uo.shape):
        if kind == "max":
            raise ValueError("zero-size array to reduction operation maximum which has no identity")
        return 0.0
    return device_norm(uo.obj, kind, weights)
