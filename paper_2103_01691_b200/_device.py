"""Device-side plumbing: column-major torch tensors, dtype codes, streams.

PyTorch is used only for device memory, streams and copies.  Tensors keep the
reference's column-major layout (tensor.py:3-6): a state of shape
(n_1, ..., n_d) is a torch tensor with strides (1, n_1, n_1*n_2, ...).  Never
call ``.contiguous()`` on a state — that would silently reorder it to C order.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from .errors import DeviceError

try:
    import torch
except ImportError:  # pragma: no cover - torch is part of the image
    torch = None

_NP_TO_CODE = {
    np.dtype(np.float32): _native.KM_F32,
    np.dtype(np.float64): _native.KM_F64,
    np.dtype(np.complex64): _native.KM_C64,
    np.dtype(np.complex128): _native.KM_C128,
}
SUPPORTED = tuple(_NP_TO_CODE)


_NP_TO_TORCH = {}
_TORCH_TO_NP = {}
if torch is not None:
    _NP_TO_TORCH = {
        np.dtype(np.float32): torch.float32,
        np.dtype(np.float64): torch.float64,
        np.dtype(np.complex64): torch.complex64,
        np.dtype(np.complex128): torch.complex128,
    }
    _TORCH_TO_NP = {
        torch.float32: np.dtype(np.float32),
        torch.float64: np.dtype(np.float64),
        torch.complex64: np.dtype(np.complex64),
        torch.complex128: np.dtype(np.complex128),
        torch.float16: np.dtype(np.float16),
        torch.int64: np.dtype(np.int64),
        torch.int32: np.dtype(np.int32),
        torch.bool: np.dtype(np.bool_),
    }


def torch_dtype(np_dtype):
    return _NP_TO_TORCH[np.dtype(np_dtype)]


def np_dtype(t_dtype):
    return _TORCH_TO_NP[t_dtype]


def code(np_dt):
    return _NP_TO_CODE[np.dtype(np_dt)]


def is_tensor(x):
    return torch is not None and isinstance(x, torch.Tensor)


def device():
    """The CUDA device used for host (numpy) inputs; raises without a GPU."""
    if torch is None or not torch.cuda.is_available():
        raise DeviceError("no CUDA device is available (this package has no CPU path)")
    return torch.device("cuda", torch.cuda.current_device())


_raw_stream = getattr(getattr(torch, "_C", None), "_cuda_getCurrentRawStream", None) if torch is not None else None


def stream_ptr(dev=None):
    """The current CUDA stream of ``dev`` as a C pointer (the fast raw-stream query when
    this torch build has it: a public ``current_stream`` lookup costs a few microseconds).

    The first time a stream is seen, a stream-K workspace is bound to it
    (:func:`_bind_stream_workspace`), so products launched on it may balance
    their last wave; the library itself never allocates device memory.
    """
    idx = None
    if _raw_stream is not None:
        idx = torch.cuda.current_device() if dev is None else (dev.index if isinstance(dev, torch.device) else int(dev))
    if idx is not None:
        raw = _raw_stream(idx)
    else:
        s = torch.cuda.current_stream(dev)
        idx, raw = s.device.index, s.cuda_stream
    if (idx, raw) not in _BOUND:
        _bind_stream_workspace(idx, raw)
    return ctypes.c_void_p(raw)


_BOUND = {}  # (device index, raw stream) -> caller-owned stream-K workspace (None: not bound)
_BOUND_MAX = 4


def _bind_stream_workspace(idx, raw):
    """Allocate (stream-ordered, on that stream) and bind the stream-K scratch of a stream.

    At most ``_BOUND_MAX`` streams per process keep one (~78 MB each on 148 SMs); the
    oldest binding is dropped first.  A dropped workspace is unbound before its memory
    returns to torch's allocator, which hands it out again only in stream order.  Streams
    being captured into a CUDA graph are not bound (graphs keep whole tiles anyway).
    """
    if torch.cuda.is_current_stream_capturing():
        return
    lib = _native.lib()
    with torch.cuda.device(idx):
        if len(_BOUND) >= _BOUND_MAX:
            (oidx, oraw), _ = next(iter(_BOUND.items()))
            with torch.cuda.device(oidx):
                _native.check(lib.km_set_stream_workspace(ctypes.c_void_p(oraw), None, 0))
            _BOUND.pop((oidx, oraw))
        nbytes = ctypes.c_size_t(0)
        _native.check(lib.km_stream_workspace_bytes(ctypes.byref(nbytes)))
        cur = torch.cuda.current_stream(idx)
        stream = cur if cur.cuda_stream == raw else torch.cuda.ExternalStream(raw, device=idx)
        with torch.cuda.stream(stream):
            ws = torch.empty(nbytes.value, dtype=torch.uint8, device=torch.device("cuda", idx))
        _native.check(lib.km_set_stream_workspace(ctypes.c_void_p(raw), ctypes.c_void_p(ws.data_ptr()),
                                                  nbytes.value))
    _BOUND[(idx, raw)] = ws


def on_device(dev):
    """Context making ``dev`` (a CUDA torch.device, or None) the current device when it is not
    already; the library's set-up caches and launches follow the current device."""
    import contextlib

    if dev is None or dev.index is None or dev.index == torch.cuda.current_device():
        return contextlib.nullcontext()
    return torch.cuda.device(dev)


def is_fortran(t):
    """Column-major dense (size-1 extents may carry any stride)."""
    s = 1
    for n, st in zip(t.shape, t.stride()):
        if n != 1 and st != s:
            return False
        s *= n
    return True


def fortran_empty(shape, dtype, dev):
    """Uninitialised column-major device tensor of the given shape."""
    shape = tuple(int(n) for n in shape)
    if not shape:
        return torch.empty((), dtype=dtype, device=dev)
    return torch.empty(tuple(reversed(shape)), dtype=dtype, device=dev).permute(
        *reversed(range(len(shape)))
    )


def as_fortran(t):
    """``t`` itself when already column-major, else a column-major copy."""
    if is_fortran(t):
        return t
    out = fortran_empty(t.shape, t.dtype, t.device)
    out.copy_(t)
    return out


def to_device(a, dtype, dev):
    """numpy array → column-major device tensor of ``dtype`` (numpy dtype).

    A page-locked source (e.g. a view of ``torch.empty(..., pin_memory=True)``)
    is copied with an asynchronous DMA on the current stream.
    """
    a = np.asarray(a)
    if a.dtype != dtype:
        a = a.astype(dtype, order="F")
    a = np.asfortranarray(a)
    if a.ndim == 0:
        return torch.tensor(a.item(), dtype=torch_dtype(dtype), device=dev)
    host = torch.from_numpy(a)  # keeps the F strides, shares memory
    if not host.is_pinned() and a.nbytes <= _STAGED_MAX:
        return upload(a, dev)  # small pageable input: staged, no stream sync
    out = fortran_empty(a.shape, torch_dtype(dtype), dev)
    out.copy_(host, non_blocking=a.nbytes >= _PINNED_MIN and host.is_pinned())
    return out


_STAGED_MAX = 16 << 20


def tensor_as(t, dtype):
    """Device tensor converted to numpy ``dtype``, keeping column-major strides."""
    td = torch_dtype(dtype)
    if t.dtype == td:
        return as_fortran(t)
    out = fortran_empty(t.shape, td, t.device)
    out.copy_(t)
    return out


def matrix_to_device(m, dtype, dev):
    """Small matrix → C-contiguous (row-major) device tensor, as the C ABI wants."""
    if is_tensor(m):
        return m.to(device=dev, dtype=torch_dtype(dtype)).contiguous()
    return upload(np.ascontiguousarray(np.asarray(m), dtype=dtype), dev)


def upload(arr, dev):
    """Host array → device tensor (same shape, strides and dtype) without a device sync.

    A copy from pageable memory waits for all earlier work on the stream
    before it starts; staging through page-locked memory instead makes
    it an asynchronous DMA, so per-step host inputs (e.g. the Magnus
    exponentials) queue behind the running products rather than stall the
    host until they finish.  The staging blocks form a small ring; a block is
    reused after the event of the copy that read it has completed (waiting
    for the oldest one when all are busy, which bounds how far the host runs
    ahead of the device).
    """
    return _upload(arr, dev)[0]


def _upload(arr, dev):
    """:func:`upload`, also returning the event of the side-stream copy (None for empty arrays)."""
    arr = np.asarray(arr)
    nbytes = arr.nbytes
    f_order = arr.ndim > 1 and arr.flags.f_contiguous and not arr.flags.c_contiguous
    if not (arr.flags.c_contiguous or f_order):
        arr = np.ascontiguousarray(arr)
    shape = arr.shape if not f_order else tuple(reversed(arr.shape))
    if nbytes == 0:
        out = torch.empty(shape, dtype=torch_dtype(arr.dtype), device=dev)
        return (out.permute(*reversed(range(arr.ndim))) if f_order else out), None
    entry = _staging_block(nbytes)
    stage = entry[0][:nbytes]
    stage.numpy()[:] = arr.ravel(order="K").view(np.uint8)
    # the copy runs on a side stream into memory allocated from that stream's pool,
    # so it overlaps the products already queued; the caller's stream waits for it
    # (event) and the tensor is marked as used there (record_stream)
    cur = torch.cuda.current_stream(dev)
    side = _upload_stream(dev)
    with torch.cuda.stream(side):
        out = torch.empty(shape, dtype=torch_dtype(arr.dtype), device=dev)
        out.view(-1).view(torch.uint8).copy_(stage, non_blocking=True)
        done = torch.cuda.Event()
        done.record(side)
    cur.wait_event(done)
    out.record_stream(cur)
    entry[1] = done
    return (out.permute(*reversed(range(arr.ndim))) if f_order else out), done


_UPLOAD_STREAMS = {}


def _upload_stream(dev):
    key = str(dev)
    if key not in _UPLOAD_STREAMS:
        _UPLOAD_STREAMS[key] = torch.cuda.Stream(dev)
    return _UPLOAD_STREAMS[key]


_STAGING = []  # ring of [pinned uint8 tensor, event of the copy that last read it (or None)]
_STAGING_SLOTS = 16
_STAGING_MIN = 1 << 20
_STAGING_AHEAD = 4  # uploads of one size in flight before the host waits


def _staging_block(nbytes):
    def touch(e):  # move to the most-recently-used end (identity, not tensor ==)
        _STAGING.pop(next(i for i, x in enumerate(_STAGING) if x is e))
        _STAGING.append(e)
        return e

    fits = [e for e in _STAGING if e[0].numel() >= nbytes]
    for e in fits:
        if e[1] is None or e[1].query():
            return touch(e)
    # all fitting blocks busy: allocate another only while few fit (pinning host memory
    # is slow and can stall the host for longer than the device work it would overlap)
    if len(fits) < _STAGING_AHEAD and (len(_STAGING) < _STAGING_SLOTS or not fits):
        if len(_STAGING) >= _STAGING_SLOTS:  # no slot is large enough: retire the oldest
            old = _STAGING.pop(0)
            if old[1] is not None:
                old[1].synchronize()
        e = [torch.empty(max(nbytes, _STAGING_MIN), dtype=torch.uint8, pin_memory=True), None]
        _STAGING.append(e)
        return e
    e = fits[0]  # all busy: wait for the least recently used one
    e[1].synchronize()
    return touch(e)


_PINNED_MIN = 1 << 20
_PINNED_POOL = []  # [pinned uint8 tensor, weakref to the ndarray handed out (or None)]
_PINNED_POOL_MAX_BYTES = 8 << 30


def pinned_host_array(shape, dtype):
    """Column-major numpy array in page-locked memory, from a small reuse pool.

    A pool buffer is handed out again only once the array returned for it (and
    therefore every numpy view of it) has been garbage-collected, so results
    returned to the caller are never overwritten.  Allocating fresh page-locked
    memory costs ~10 ms per 256 MB; the pool makes repeated drop-in calls pay it
    once.
    """
    import weakref

    dtype = np.dtype(dtype)
    nbytes = int(np.prod(shape, dtype=np.int64)) * dtype.itemsize
    entry = None
    for e in _PINNED_POOL:
        if e[0].numel() == nbytes and (e[1] is None or e[1]() is None):
            entry = e
            break
    if entry is None:
        buf = torch.empty(max(nbytes, 1), dtype=torch.uint8, pin_memory=True)
        entry = [buf, None]
        if sum(e[0].numel() for e in _PINNED_POOL) + nbytes <= _PINNED_POOL_MAX_BYTES:
            _PINNED_POOL.append(entry)
    arr = entry[0][:nbytes].numpy().view(dtype).reshape(tuple(shape), order="F")
    entry[1] = weakref.ref(_owner(arr))
    return arr


def _owner(arr):
    """The object at the end of ``arr``'s base chain (here the torch tensor behind ``.numpy()``).

    numpy collapses view bases: ``arr[..., 0]``, ``arr.real`` or ``arr.T`` reference this
    terminal object, not ``arr`` itself, so it is alive exactly as long as any view of the
    buffer is.  A weakref to ``arr`` would die while such views still read the buffer.
    """
    base = arr
    while isinstance(base, np.ndarray) and base.base is not None:
        base = base.base
    return base


def to_host(t):
    """Device tensor → numpy array with the same (column-major) layout.

    Large results land in page-locked memory (see :func:`pinned_host_array`)
    so the device→host copy runs at DMA speed.
    """
    t = t.detach()
    if t.is_cuda and t.numel() * t.element_size() >= _PINNED_MIN and is_fortran(t):
        arr = pinned_host_array(tuple(t.shape), np_dtype(t.dtype))
        host = torch.from_numpy(arr.reshape(-1, order="F"))
        src = t.permute(*reversed(range(t.dim()))).reshape(-1)
        host.copy_(src, non_blocking=True)
        torch.cuda.current_stream(t.device).synchronize()
        return arr
    return t.cpu().numpy()


_VEC_CACHE = {}
_VEC_CACHE_MAX = 64

try:
    _libc_memcmp = ctypes.CDLL(None).memcmp
    _libc_memcmp.restype = ctypes.c_int
    _libc_memcmp.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t]
except (OSError, AttributeError):  # pragma: no cover - every Linux libc has memcmp
    _libc_memcmp = None


def _same_bytes(a, b):
    """Byte equality of two arrays with the same dtype, shape and memory order."""
    if a.nbytes == 0:
        return True
    if _libc_memcmp is not None:
        return _libc_memcmp(a.ctypes.data, b.ctypes.data, a.nbytes) == 0
    return np.array_equal(a.reshape(-1, order="K").view(np.uint8), b.reshape(-1, order="K").view(np.uint8))


def cached_vector(v, dtype, dev):
    """Device copy of a small host vector/matrix, memoised per host buffer.

    The entry is keyed by the host buffer (address, dtype, shape, strides) and
    validated on every hit with a memcmp against a snapshot taken at upload, so
    an array modified in place (or a new array at a recycled address) is
    uploaded again.  A memcmp reads the matrix once; hashing its bytes, the
    previous key, cost ~6x more host time per call (1 ms for a 512 x 512
    complex64 factor, on the critical path of every mu_mode_product call).
    """
    if is_tensor(v):
        if v.device == dev and v.dtype == torch_dtype(dtype) and v.is_contiguous():
            return v
        return v.to(device=dev, dtype=torch_dtype(dtype)).contiguous()
    src = np.asarray(v)
    if not (src.flags.c_contiguous or src.flags.f_contiguous):
        src = np.ascontiguousarray(src)
    key = (str(dev), np.dtype(dtype).str, src.dtype.str, src.shape, src.strides, src.ctypes.data)
    hit = _VEC_CACHE.get(key)
    if hit is not None and _same_bytes(hit[0], src):
        # the upload ran on a side stream and only the stream current at upload time waited
        # for it: order this hit's stream after the copy too (free once it has completed)
        if hit[2] is not None and stream_ptr(dev).value != hit[3]:
            cur = torch.cuda.current_stream(dev)
            cur.wait_event(hit[2])
            hit[1].record_stream(cur)
        return hit[1]
    t, ev = _upload(np.ascontiguousarray(src, dtype=dtype), dev)
    if hit is None and len(_VEC_CACHE) >= _VEC_CACHE_MAX:
        _VEC_CACHE.pop(next(iter(_VEC_CACHE)))
    _VEC_CACHE[key] = (src.copy(order="K"), t, ev, stream_ptr(dev).value)
    return t
