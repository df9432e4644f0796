"""Host-pipelined Tucker operator for numpy (host) inputs.

A drop-in call such as ``step(cache, u_numpy)`` has to move the state to the
device and the result back: 2 x 268 MB over PCIe at n=256^3 c128, about 3x
the device compute.  This driver hides the compute under the copies:

* the state is cut into C slabs along the LAST direction d, which are
  contiguous in the column-major host array;
* slab c goes host→device on a copy stream while the compute stream runs the
  products of directions 1..d-1 on slab c-1 (those never mix slabs);
* the direction-d product is then launched in C row blocks of E_d
  (a row block of a row-major matrix is contiguous), each producing one
  contiguous output slab, which goes device→host on a second copy stream
  while the next block is computed.

Pointwise ops (the splitting phases) see each slab as a tensor of its own:
their index arithmetic is local, so the direction-d weight/diagonal pointer is
offset to the slab's first index.  Results are identical to the unpipelined
``km_tucker`` path (same kernels, same per-element arithmetic).
"""

from __future__ import annotations

import ctypes
import time
from math import prod

import numpy as np

from . import _device as dv
from . import _native

MIN_BYTES = 16 << 20
FIB_PIECES = 4
TAIL_SHIFTS = (3, 4, 5, 6)  # last input slabs: n/8, n/16, n/32, n/64
_streams = {}
TRACE = []  # (label, event, host time) of the last call when tracing is on (tools/e2e_timeline.py)
_trace_on = False


def _side_streams(dev):
    key = str(dev)
    if key not in _streams:
        _streams[key] = (dv.torch.cuda.Stream(dev), dv.torch.cuda.Stream(dev))
    return _streams[key]


def _chunks(n, parts):
    parts = max(1, min(parts, n))
    base, extra = divmod(n, parts)
    out, start = [], 0
    for i in range(parts):
        size = base + (1 if i < extra else 0)
        out.append((start, size))
        start += size
    return out


def _input_slabs(n, parts):
    """Slabs along the last direction for the host-to-device phase.

    A slab's products (directions 1..d-1) take about half as long as its copy
    (tools/e2e_timeline.py: 0.33 against 0.67 ms for 36 of 256 planes), so the
    last slabs shrink geometrically (n/8, n/16, n/32, n/64): each one's products
    finish while the next, half-size slab is still in flight, and only the
    smallest slab's products remain when the copies end.  The rest is uniform.
    """
    if parts < len(TAIL_SHIFTS) + 2 or n < 16 * parts:
        return _chunks(n, parts)
    tail = [max(1, n >> s) for s in TAIL_SHIFTS]
    head = _chunks(n - sum(tail), parts - len(tail))
    out, start = list(head), n - sum(tail)
    for size in tail:
        out.append((start, size))
        start += size
    return out


# Pageable (ordinary numpy) inputs: a cudaMemcpy from pageable memory stages through the
# driver's own small pinned buffers at ~10-20 GB/s and blocks the host per slab (the
# drop-in step at 256^3 ran at 34 steps/s against 101 with a pinned input).  Instead the
# input is copied by several host threads (numpy copies release the GIL) into a ring of
# page-locked staging blocks, each shipped by an asynchronous DMA as soon as it is full,
# so the host copy of block k+1 overlaps the DMA of block k.
STAGE_BYTES = 32 << 20
STAGE_BLOCKS = 3
_stage_ring = {}  # device -> list of [pinned uint8 tensor, event of the DMA that read it]
_copy_pool = None


def _copy_threads():
    global _copy_pool
    if _copy_pool is None:
        import os
        from concurrent.futures import ThreadPoolExecutor

        _copy_pool = ThreadPoolExecutor(max_workers=max(1, min(8, (os.cpu_count() or 2) // 2)))
    return _copy_pool


def _parallel_copy(dst, src):
    """dst[...] = src for equal-size contiguous 1-D arrays, split over the copy threads."""
    pool = _copy_threads()
    n = src.size
    parts = pool._max_workers if n * src.itemsize >= (4 << 20) else 1
    if parts == 1:
        np.copyto(dst, src)
        return
    cuts = [n * i // parts for i in range(parts + 1)]
    list(pool.map(lambda i: np.copyto(dst[cuts[i]:cuts[i + 1]], src[cuts[i]:cuts[i + 1]]), range(parts)))


def _staging(dev):
    key = str(dev)
    ring = _stage_ring.get(key)
    if ring is None:
        ring = [[dv.torch.empty(STAGE_BYTES, dtype=dv.torch.uint8, pin_memory=True), None]
                for _ in range(STAGE_BLOCKS)]
        _stage_ring[key] = ring
    return ring


def _staged_h2d(dst_flat, src_np, lo, hi, stream, dev):
    """dst_flat[lo:hi] = src_np[lo:hi] (1-D element ranges) through the pinned staging ring,
    DMA on ``stream``; returns the event of the last DMA."""
    torch = dv.torch
    ring = _staging(dev)
    es = src_np.itemsize
    per = STAGE_BYTES // es
    ev = None
    k = 0
    for a in range(lo, hi, per):
        b = min(hi, a + per)
        blk = ring[k % len(ring)]
        k += 1
        if blk[1] is not None:
            blk[1].synchronize()  # the DMA that last read this block is done
        stage = blk[0][: (b - a) * es].numpy().view(src_np.dtype)
        _parallel_copy(stage, src_np[a:b])
        ev = torch.cuda.Event()
        with torch.cuda.stream(stream):
            dst_flat[a:b].copy_(torch.from_numpy(stage), non_blocking=True)  # page-locked source: async DMA
            ev.record(stream)
        blk[1] = ev
    return ev


def eligible(host, d):
    return 2 <= d <= _native.MAX_D and host.nbytes >= MIN_BYTES


def _op_for_slab(op, dims, last, start, size):
    """Copy of a pointwise op restricted to the slab [start, start+size) of the last direction."""
    if op is None:
        return None
    o = _native.PointOp()
    ctypes.pointer(o)[0] = op
    o.d = len(dims)
    for i, n in enumerate(dims):
        o.dims[i] = n
    o.dims[last] = size
    if op.kind == _native.OP_GPE_PHASE:
        o.weights[last] = op.weights[last] + 8 * start  # f64 vector
    elif op.kind == _native.OP_DIAG and op.diag_dir == last:
        o.diag = op.diag + 16 * start  # c128 vector
    return o


def _mark(label, stream):
    if _trace_on:
        ev = dv.torch.cuda.Event(enable_timing=True)
        ev.record(stream)
        TRACE.append((label, ev, time.perf_counter()))


def tucker_host_pipelined(host, u_dt, mats_dev, codes, rows, pre, post, out_shape, cdt, dev, parts=8):
    """``post(pre(host) x_1 mats[0] ... x_d mats[d-1])`` for a host array; returns a host array.

    ``host`` is column-major of numpy dtype ``u_dt`` (complex when ``pre`` or
    ``post`` is given); ``mats_dev`` are row-major device matrices (None =
    skip) with dtype codes ``codes``; ``cdt`` is the result dtype.
    """
    torch = dv.torch
    lib = _native.lib()
    d = host.ndim
    dims = tuple(host.shape)
    last = d - 1
    compute = torch.cuda.current_stream(dev)
    s_in, s_out = _side_streams(dev)
    stream_c = dv.stream_ptr(dev)  # the compute stream (binds its stream-K workspace once)
    slabs = _input_slabs(dims[last], parts)
    max_slab = max(sz for _, sz in slabs)
    inner = prod(dims[:last])
    u_dt = np.dtype(u_dt)

    # the input copies go first: they are the critical path, so a page-locked input
    # is queued on the copy stream before the rest of the set-up (~0.08 ms of host
    # work).  The input buffer comes from the copy stream's own allocator pool and is
    # marked as used by the compute stream, so the copies need not wait for unrelated
    # work the caller queued on the compute stream.
    if _trace_on:
        TRACE.clear()
        _mark("start", compute)
    with torch.cuda.stream(s_in):
        src_all = torch.empty(host.size, dtype=dv.torch_dtype(u_dt), device=dev)
    src_all.record_stream(compute)
    h_t = torch.from_numpy(host.reshape(-1, order="F"))
    pinned_in = h_t.is_pinned()

    def h2d(start, size):
        lo, hi = inner * start, inner * (start + size)
        ev = torch.cuda.Event()
        with torch.cuda.stream(s_in):
            src_all[lo:hi].copy_(h_t[lo:hi], non_blocking=pinned_in)
            ev.record(s_in)
            _mark(f"h2d slab {start}+{size}", s_in)
        return ev

    host_flat = host.reshape(-1, order="F")

    def h2d_staged(start, size):
        lo, hi = inner * start, inner * (start + size)
        ev = _staged_h2d(src_all, host_flat, lo, hi, s_in, dev)
        _mark(f"h2d staged slab {start}+{size}", s_in)
        return ev

    h2d_done = [h2d(start, size) for (start, size) in slabs] if pinned_in else None
    pre_active = [i for i in range(last) if mats_dev[i] is not None]
    has_last = mats_dev[last] is not None

    # dtype / shape walk of one slab through directions 1..d-1
    walk, shape, dt = [], list(dims[:last]) + [max_slab], u_dt
    for mu in pre_active:
        dt = np.result_type(dt, _code_dtype(codes[mu]))
        shape = list(shape)
        shape[mu] = rows[mu]
        walk.append((mu, dt, prod(shape)))
    mid_dt = dt
    mid_shape = tuple(shape[:last]) + (dims[last],)
    inner_mid = prod(mid_shape[:last])
    ws_bytes = max([inner * max_slab * u_dt.itemsize] + [n * t.itemsize for _, t, n in walk])
    ws = [torch.empty(ws_bytes, dtype=torch.uint8, device=dev) for _ in range(2)]

    def view(buf, n, npdt):
        return buf[: n * np.dtype(npdt).itemsize].view(dv.torch_dtype(npdt))

    direct_mid = has_last and not pre_active and pre is None
    mid_all = None
    if has_last:
        mid_all = src_all if direct_mid else torch.empty(prod(mid_shape), dtype=dv.torch_dtype(mid_dt), device=dev)
    out_dev = torch.empty(prod(out_shape), dtype=dv.torch_dtype(cdt), device=dev)
    inner_out = prod(out_shape[:last])

    host_arr = dv.pinned_host_array(out_shape, cdt)
    host_out_flat = torch.from_numpy(host_arr.reshape(-1, order="F"))

    def ship(lo, hi):
        ev = torch.cuda.Event()
        ev.record(compute)
        s_out.wait_event(ev)
        with torch.cuda.stream(s_out):
            host_out_flat[lo:hi].copy_(out_dev[lo:hi], non_blocking=True)
            _mark(f"d2h {lo}", s_out)

    from .tensor import launch_product

    def product(src, sdt, mu, m, shape, dst, op, lptr=None):
        nl, nr = prod(shape[:mu]), prod(shape[mu + 1:])
        lp = mats_dev[mu].data_ptr() if lptr is None else lptr
        launch_product(src.data_ptr(), dv.code(sdt), lp, codes[mu], dst.data_ptr(), m, nl, shape[mu], nr, op,
                       stream_c, dev)

    # ---- phase 1: per input slab: H2D, pre op, directions 1..d-1
    for k, (start, size) in enumerate(slabs):
        lo, hi = inner * start, inner * (start + size)
        # a pageable input is staged slab by slab here (host threads + DMA), just ahead of its products
        compute.wait_event(h2d_done[k] if h2d_done is not None else h2d_staged(start, size))
        cur, cdtype = src_all[lo:hi], u_dt
        shape = list(dims[:last]) + [size]
        final_here = not has_last
        if pre is not None:
            dst = view(ws[0], cur.numel(), cdtype) if (pre_active or has_last) else out_dev[lo:hi]
            if final_here and not pre_active:
                dst = out_dev[inner_out * start: inner_out * start + cur.numel()]
            op = _op_for_slab(pre, shape, last, start, size)
            _native.check(lib.km_pointwise(cur.data_ptr(), dst.data_ptr(), dv.code(cdtype), cur.numel(),
                                           ctypes.byref(op), stream_c))
            cur = dst
        for idx, (mu, ndt, _) in enumerate(walk):
            new_shape = list(shape)
            new_shape[mu] = rows[mu]
            n_new = prod(new_shape)
            last_pre = idx == len(walk) - 1
            if last_pre and has_last:
                dst = mid_all[inner_mid * start: inner_mid * start + n_new]
            elif last_pre:
                dst = out_dev[inner_out * start: inner_out * start + n_new]
            else:
                dst = view(ws[(idx + 1) % 2], n_new, ndt)
            op = _op_for_slab(post, new_shape, last, start, size) if (last_pre and final_here) else None
            product(cur, cdtype, mu, rows[mu], shape, dst, op)
            _mark(f"dir {mu + 1} slab {start}", compute)
            cur, cdtype, shape = dst, ndt, new_shape
        if has_last and not walk and not direct_mid:
            mid_all[inner_mid * start: inner_mid * start + cur.numel()].copy_(cur)
        if final_here:
            olo = inner_out * start
            if not walk:
                if pre is None:
                    out_dev[olo: olo + cur.numel()].copy_(cur)
                if post is not None:
                    seg = out_dev[olo: olo + cur.numel()]
                    op = _op_for_slab(post, shape, last, start, size)
                    _native.check(lib.km_pointwise(seg.data_ptr(), seg.data_ptr(), dv.code(cdt), seg.numel(),
                                                   ctypes.byref(op), stream_c))
            ship(olo, olo + inner_out * size)

    # ---- phase 2: direction d in row blocks of E_d; each output slab D2H as it completes
    if has_last:
        row_bytes = dims[last] * _code_dtype(codes[last]).itemsize
        # row blocks of whole 64-row output tiles, so no launch pays for a padded tile
        parts2 = max(1, min(parts, rows[last] // 64)) if rows[last] >= 64 else 1
        blocks = _chunks(rows[last], parts2)
        # the first row block in FIB_PIECES fiber pieces (km_mumode_fibers), each shipped
        # as a strided 2-D copy: the device-to-host copies start after ~1/FIB_PIECES of
        # the block instead of all of it (256^3: 0.26 -> ~0.08 ms between the last H2D
        # copy and the first D2H copy); double precision, no fused op
        es_out = np.dtype(cdt).itemsize
        piece = inner_mid // FIB_PIECES
        double = (np.dtype(mid_dt) in (np.dtype(np.float64), np.dtype(np.complex128))
                  and codes[last] in (_native.KM_F64, _native.KM_C128))
        if (post is None and double and len(blocks) > 1 and inner_mid == inner_out
                and inner_mid % FIB_PIECES == 0 and piece % 128 == 0):
            start, size = blocks.pop(0)
            lp = mats_dev[last].data_ptr() + start * row_bytes
            for c in range(FIB_PIECES):
                f0 = c * piece
                _native.check(lib.km_mumode_fibers(mid_all.data_ptr(), dv.code(mid_dt), lp, codes[last],
                                                   out_dev[inner_out * start:].data_ptr(), size, inner_mid,
                                                   dims[last], f0, piece, stream_c))
                _mark(f"dir {last + 1} rows {start}+{size} fibers {f0}+{piece}", compute)
                ev = torch.cuda.Event()
                ev.record(compute)
                s_out.wait_event(ev)
                off = (inner_out * start + f0) * es_out
                _native.check(lib.km_copy_2d(host_out_flat.data_ptr() + off, inner_out * es_out,
                                             out_dev.data_ptr() + off, inner_out * es_out, piece * es_out, size,
                                             ctypes.c_void_p(s_out.cuda_stream)))
                _mark(f"d2h rows {start} fibers {f0}", s_out)
        for (start, size) in blocks:
            olo = inner_out * start
            dst = out_dev[olo: olo + inner_out * size]
            op = _op_for_slab(post, list(out_shape[:last]) + [size], last, start, size)
            product(mid_all, mid_dt, last, size, list(mid_shape), dst, op,
                    lptr=mats_dev[last].data_ptr() + start * row_bytes)
            _mark(f"dir {last + 1} rows {start}+{size}", compute)
            ship(olo, olo + inner_out * size)
    s_out.synchronize()
    return host_arr


def _code_dtype(code):
    return {_native.KM_F32: np.dtype(np.float32), _native.KM_F64: np.dtype(np.float64),
            _native.KM_C64: np.dtype(np.complex64), _native.KM_C128: np.dtype(np.complex128)}[code]
