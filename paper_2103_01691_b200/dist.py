"""Steppers that keep the state resident on the device(s) across steps.

* :class:`LocalStepper` — one GPU.  The exact step ``u x_1 E_1 ... x_d E_d``
  runs as one ``km_tucker`` call per step over three device buffers (state,
  one scratch, next state; the next-state buffer doubles as the second
  scratch): the reference's acceptance criterion 9 bound of 3x the state
  (test_acceptance.py:298-321) holds on the device.
* :class:`SlabStepper` — several GPUs, one process per GPU (torch.distributed
  over NCCL).  See the class docstring.
"""

from __future__ import annotations

import ctypes
from math import prod

import numpy as np

from . import _device as dv
from . import _native


class LocalStepper:
    """Repeated exact steps of a device-resident column-major state on one GPU."""

    def __init__(self, state, mats, pre=None, post=None):
        self.torch = dv.torch
        self.a = state
        self.b = dv.torch.empty_like(state)
        self.w = dv.torch.empty_like(state)
        self.mats = list(mats)
        self.dims = tuple(state.shape)
        self.d = len(self.dims)
        self.code = dv.code(dv.np_dtype(state.dtype))
        self._c_dims = (ctypes.c_int64 * self.d)(*self.dims)
        self._c_mats = (ctypes.c_void_p * self.d)(*[m.data_ptr() for m in self.mats])
        self._c_codes = (ctypes.c_int * self.d)(*[dv.code(dv.np_dtype(m.dtype)) for m in self.mats])
        self._c_rows = (ctypes.c_int64 * self.d)(*[m.shape[0] for m in self.mats])
        self.pre, self.post = pre, post
        self.launches_per_step = self.d + (1 if pre is not None else 0) - \
            (1 if _native.plane_fused(self.code, self.dims, list(self._c_codes), list(self._c_rows)) else 0)
        self.lib = _native.lib()

    def step(self):
        """``a <- a x_1 E_1 ... x_d E_d``; the output buffer doubles as the second scratch."""
        stream = dv.stream_ptr(self.a.device)
        _native.check(self.lib.km_tucker(
            self.a.data_ptr(), self.code, self.d, self._c_dims, self._c_mats, self._c_codes, self._c_rows,
            self.b.data_ptr(), self.w.data_ptr(), None,
            None if self.pre is None else ctypes.byref(self.pre),
            None if self.post is None else ctypes.byref(self.post), stream))
        self.a, self.b = self.b, self.a

    def run(self, steps, persistent=False, paired=None):
        """``steps`` exact steps.

        Small complex128 cubes (extents 32, 48 or 64, square complex128 factors, no phase ops)
        take ``km_steps_paired`` by default (``paired=None``): every two steps as three fused
        launches, (1,2) per i3-plane, the two steps' direction-3 products together per block
        of fibers, (1,2) again; ``paired=False`` keeps one ``km_tucker``
        launch per step.  ``persistent=True`` runs them instead as ONE launch (``km_steps_small``: the 3·steps
        sweeps as a dataflow of 32 x 32 tiles with dependency counters) for complex128 3D
        states whose extents are multiples of 32 up to 96.  It is correct and kept for the
        record, but measured slower than the per-step launches replayed as a CUDA graph
        (64³ x 10 steps: 0.29-0.31 ms against 0.227 ms): a consumer tile of
        the next sweep reads the output of ~all tiles of the previous one, so the sweeps
        serialise on the tile latency (staging + MMA + publish), which exceeds a launch gap.
        """
        if steps < 1:
            return
        if not persistent and paired is not False and self.paired_ok():
            _native.check(self.lib.km_steps_paired(
                self.a.data_ptr(), self.mats[0].data_ptr(), self.mats[1].data_ptr(), self.mats[2].data_ptr(),
                *self.dims, steps, self.b.data_ptr(), self.w.data_ptr(), dv.stream_ptr(self.a.device)))
            self.a, self.b = self.b, self.a
            return
        ws = self._steps_workspace(steps) if persistent else None
        if ws is None:
            for _ in range(steps):
                self.step()
            return
        _native.check(self.lib.km_steps_small(
            self.a.data_ptr(), self.mats[0].data_ptr(), self.mats[1].data_ptr(), self.mats[2].data_ptr(),
            *self.dims, steps, ws.data_ptr(), ws.numel(), dv.stream_ptr(self.a.device)))

    def paired_ok(self):
        """Whether ``run`` takes ``km_steps_paired`` (its shape and dtype rules)."""
        torch = self.torch
        return (self.d == 3 and self.pre is None and self.post is None and self.a.dtype == torch.complex128
                and dv.is_fortran(self.a) and all(n in _native.PLANE_EXTENTS for n in self.dims)
                and all(m.dtype == torch.complex128 and tuple(m.shape) == (n, n) and m.is_contiguous()
                        for m, n in zip(self.mats, self.dims)))

    def launches_for(self, steps):
        """Launches ``run(steps)`` issues (the bench's ``gpu_launches``)."""
        if self.paired_ok():
            return (steps // 2) * 3 + (steps % 2) * 2
        return steps * self.launches_per_step

    def _steps_workspace(self, steps):
        torch = self.torch
        if (self.d != 3 or self.pre is not None or self.post is not None or self.a.dtype != torch.complex128
                or not dv.is_fortran(self.a)
                or any(m.dtype != torch.complex128 or tuple(m.shape) != (n, n) for m, n in zip(self.mats, self.dims))):
            return None
        nbytes = ctypes.c_size_t(0)
        if self.lib.km_steps_small_workspace_bytes(*self.dims, steps, ctypes.byref(nbytes)) != _native.KM_OK:
            return None
        if getattr(self, "_small_ws", None) is None or self._small_ws.numel() < nbytes.value:
            self._small_ws = torch.empty(nbytes.value, dtype=torch.uint8, device=self.a.device)
        return self._small_ws

    @property
    def state(self):
        return self.a

    def time_launches(self, reps=10):
        """Mean device time (ms) of each direction's product launch, CUDA events on the launch stream."""
        torch = self.torch
        stream = torch.cuda.current_stream(self.a.device)
        out = []
        for mu in range(self.d):
            nl, nr = prod(self.dims[:mu]), prod(self.dims[mu + 1:])
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            call = lambda: _native.check(self.lib.km_mumode(  # noqa: E731
                self.a.data_ptr(), self.code, self.mats[mu].data_ptr(), self._c_codes[mu], self.w.data_ptr(),
                self._c_rows[mu], nl, self.dims[mu], nr, None, ctypes.c_void_p(stream.cuda_stream)))
            call()
            ev0.record(stream)
            for _ in range(reps):
                call()
            ev1.record(stream)
            ev1.synchronize()
            out.append(ev0.elapsed_time(ev1) / reps)
        return out


class Prod:
    """One product of a slab schedule: direction ``mu`` with matrix ``mat`` (a key of the
    stepper's matrices: "E1", "E2", "E3", "E3p0", "E3p1", "E3r0", "E3r1") of ``m`` rows, the
    (n_left, n_mu, n_right) flattening, the blocked input / output (km_mumode_split) and the
    source / destination buffers ("a", "w", "send", "recv") with element offsets."""

    __slots__ = ("mu", "mat", "m", "nl", "nmu", "nr", "kcb", "kbs", "ncb", "nbs", "src", "soff", "dst", "doff",
                 "acc")

    def __init__(self, mu, mat, m, nl, nmu, nr, kcb, kbs, ncb, nbs, src, soff, dst, doff, acc=0):
        self.mu, self.mat, self.m, self.nl, self.nmu, self.nr = mu, mat, m, nl, nmu, nr
        self.kcb, self.kbs, self.ncb, self.nbs = kcb, kbs, ncb, nbs
        self.src, self.soff, self.dst, self.doff = src, soff, dst, doff
        self.acc = acc  # 1: accumulate into the destination (km_mumode_split accumulate)

    def plain_out(self):
        return self.ncb == self.m


class SlabPlan:
    """Index bookkeeping of the slab decomposition of a 3D state over P ranks.

    Layout "A": rank r holds ``u[:, :, r*c3:(r+1)*c3]`` as a column-major
    (n1, n2, c3) array (c3 = n3/P).  Layout "B": rank r holds
    ``u[:, r*c2:(r+1)*c2, :]`` as (n1, c2, n3) (c2 = n2/P).  Both are
    contiguous slices of the global column-major array's index space along
    one direction, so scatter/gather need no reordering of elements inside a
    slab.  The all-to-all moves blocks of n1*c2*c3 elements:

    * A -> B: rank r sends to rank s the (n1, c2, c3) block with i2 in s's
      chunk.  The direction-2 product writes its output directly in that
      per-peer block order (``out_block = c2``), so the send buffer needs no
      pack pass; the receive buffer, blocks ordered by source rank = i3 chunk,
      IS the layout-B slab.
    * B -> A: the send buffer is the layout-B slab itself (the block for peer
      s is the contiguous i3-chunk of s); the receive buffer holds blocks
      ordered by source rank = i2 chunk, which the next direction-2 product
      reads in place (``in_block = c2``), so no unpack pass either.
    """

    def __init__(self, dims, nranks):
        if len(dims) != 3:
            raise ValueError("the slab decomposition is implemented for 3D states")
        n1, n2, n3 = (int(x) for x in dims)
        if n2 % nranks or n3 % nranks:
            raise ValueError(f"extents {dims} do not split evenly over {nranks} ranks")
        self.dims = (n1, n2, n3)
        self.P = nranks
        self.c2, self.c3 = n2 // nranks, n3 // nranks
        self.shape_a = (n1, n2, self.c3)
        self.shape_b = (n1, self.c2, n3)
        self.block = n1 * self.c2 * self.c3
        self.local = n1 * n2 * self.c3

    def slab_a(self, u, rank):
        return u[:, :, rank * self.c3:(rank + 1) * self.c3]

    def slab_b(self, u, rank):
        return u[:, rank * self.c2:(rank + 1) * self.c2, :]

    def overlap_ok(self):
        """The two-half schedule needs half-chunks of direction 3 that the blocked loaders take:
        c3/2 a multiple of 16 (input blocks) and c2 a multiple of 16."""
        return self.c3 % 32 == 0 and self.c2 % 16 == 0

    def schedule(self, layout, overlap):
        """One step from ``layout``: (pre, post, exchange), each pre/post a list of groups of
        products :class:`Prod`; exchange ``h`` moves ``size`` elements at offset ``h * size`` of
        the send / receive buffers after pre group ``h``; post group ``h`` reads only what
        exchanges ``0..h`` delivered.

        Serial (``overlap`` False): the schedule of :meth:`even_calls` / :meth:`odd_calls`, one
        exchange of the whole slab.  Overlapped: the last product before the exchange runs in
        two halves, each followed by its own all-to-all, so half 0 moves while half 1 computes:

        * even (A -> B): direction 2 on the i3-halves of the slab (n_right = c3/2), per-peer
          blocks of (n1, c2, c3/2); the receive buffer holds block (h, source q) at
          ``(h*P + q) * bs/2``.  Direction 3 contracts over i3, so it splits the same way:
          half h of its sum reads receive half h as a blocked input (in_block = c3/2) against
          the matching columns of E3 (``E3p0`` / ``E3p1``), the second half accumulating into
          the first's output — half 0's part runs while half 1 is still moving;
        * odd (B -> A): direction 1, then direction 3 in two halves of output rows (``E3r0`` /
          ``E3r1``: the rows of E3 whose i3 lie in the first / second half of every peer's
          chunk), per-peer blocks of (n1, c2, c3/2); direction 2 then runs per half (i3 of
          the half = its n_right) as soon as that half has arrived.
        """
        n1, n2, n3 = self.dims
        c2, c3, bs, P = self.c2, self.c3, self.block, self.P
        if not overlap:
            if layout == "A":
                pre = [[Prod(0, "E1", n1, 1, n1, n2 * c3, n1, 0, n1, 0, "a", 0, "w", 0),
                        Prod(1, "E2", n2, n1, n2, c3, n2, 0, c2, bs, "w", 0, "send", 0)]]
                post = [[Prod(2, "E3", n3, n1 * c2, n3, 1, n3, 0, n3, 0, "recv", 0, "a", 0)]]
            else:
                pre = [[Prod(2, "E3", n3, n1 * c2, n3, 1, n3, 0, n3, 0, "a", 0, "w", 0),
                        Prod(0, "E1", n1, 1, n1, c2 * n3, n1, 0, n1, 0, "w", 0, "send", 0)]]
                post = [[Prod(1, "E2", n2, n1, n2, c3, c2, bs, n2, 0, "recv", 0, "a", 0)]]
            return pre, post, P * bs
        h3, bsh = c3 // 2, bs // 2
        if layout == "A":
            pre = [[Prod(0, "E1", n1, 1, n1, n2 * c3, n1, 0, n1, 0, "a", 0, "w", 0),
                    Prod(1, "E2", n2, n1, n2, h3, n2, 0, c2, bsh, "w", 0, "send", 0)],
                   [Prod(1, "E2", n2, n1, n2, h3, n2, 0, c2, bsh, "w", n1 * n2 * h3, "send", P * bsh)]]
            post = [[Prod(2, "E3p0", n3, n1 * c2, n3 // 2, 1, h3, bsh, n3, 0, "recv", 0, "a", 0)],
                    [Prod(2, "E3p1", n3, n1 * c2, n3 // 2, 1, h3, bsh, n3, 0, "recv", P * bsh, "a", 0, acc=1)]]
        else:
            pre = [[Prod(0, "E1", n1, 1, n1, c2 * n3, n1, 0, n1, 0, "a", 0, "w", 0),
                    Prod(2, "E3r0", n3 // 2, n1 * c2, n3, 1, n3, 0, h3, bsh, "w", 0, "send", 0)],
                   [Prod(2, "E3r1", n3 // 2, n1 * c2, n3, 1, n3, 0, h3, bsh, "w", 0, "send", P * bsh)]]
            post = [[Prod(1, "E2", n2, n1, n2, h3, c2, bsh, n2, 0, "recv", 0, "a", 0)],
                    [Prod(1, "E2", n2, n1, n2, h3, c2, bsh, n2, 0, "recv", P * bsh, "a", n1 * n2 * h3)]]
        return pre, post, P * bsh

    def e3_column_halves(self):
        """pi_h: column k' of E3p<h> is column pi_h[k'] of E3 (the even-step receive order of half h)."""
        P, c3, h3 = self.P, self.c3, self.c3 // 2
        return [np.array([q * c3 + h * h3 + j for q in range(P) for j in range(h3)]) for h in range(2)]

    def e3_row_halves(self):
        """rho_g: row i' of E3r<g> is row rho_g[i'] of E3 (the odd-step send order)."""
        P, c3, h3 = self.P, self.c3, self.c3 // 2
        return [np.array([q * c3 + g * h3 + j for q in range(P) for j in range(h3)]) for g in range(2)]

    # product calls: (direction index, m, n_left, n_mu, n_right, in_block, in_stride, out_block, out_stride)
    def even_calls(self):
        """Layout A: directions 1, 2 (packed output) | exchange | direction 3 in layout B."""
        n1, n2, n3 = self.dims
        c2, c3, bs = self.c2, self.c3, self.block
        before = [(0, n1, 1, n1, n2 * c3, n1, 0, n1, 0),
                  (1, n2, n1, n2, c3, n2, 0, c2, bs)]
        after = [(2, n3, n1 * c2, n3, 1, n3, 0, n3, 0)]
        return before, after

    def odd_calls(self):
        """Layout B: directions 3, 1 | exchange | direction 2 reading blocked input, into layout A."""
        n1, n2, n3 = self.dims
        c2, c3, bs = self.c2, self.c3, self.block
        before = [(2, n3, n1 * c2, n3, 1, n3, 0, n3, 0),
                  (0, n1, 1, n1, c2 * n3, n1, 0, n1, 0)]
        after = [(1, n2, n1, n2, c3, c2, bs, n2, 0)]
        return before, after


class SlabStepper:
    """Exact steps of a 3D state split into slabs over the ranks of a process group.

    One process per GPU; ``comm`` moves the per-peer blocks (NCCL
    ``all_to_all_single`` over NVLink, see :class:`NcclExchange`).  Because
    the factors commute, consecutive steps alternate the direction order
    ({1,2} | a2a | {3}, then {3,1} | a2a | {2}) so that every step needs ONE
    exchange; the pack/unpack are fused into the direction-2 product (see
    :class:`SlabPlan`).  After an odd number of steps the state is in layout
    B, after an even number in layout A (``self.layout``).
    """

    def __init__(self, plan, rank, local_a, mats, comm, overlap=True):
        torch = dv.torch
        self.plan, self.rank, self.comm = plan, rank, comm
        self.mats = list(mats)
        n = plan.local
        self.a = local_a.reshape(-1) if local_a.dim() > 1 else local_a
        if self.a.numel() != n:
            raise ValueError("local slab has the wrong size")
        self.w = torch.empty_like(self.a)
        self.send = torch.empty_like(self.a)
        self.recv = torch.empty_like(self.a)
        self.layout = "A"
        self.code = dv.code(dv.np_dtype(self.a.dtype))
        self.mcodes = [dv.code(dv.np_dtype(m.dtype)) for m in self.mats]
        self.lib = _native.lib()
        self.overlap = bool(overlap) and plan.overlap_ok()
        self.derived = {}
        if self.overlap:
            self._derive(self.mats[2])
        self.launches_per_step = 5 if self.overlap else 3
        self._works = []

    def _derive(self, e3):
        """E3's two column halves in the even-step receive order and its two row halves in the
        odd-step send order (contiguous row-major copies, as the kernels read factors)."""
        torch = dv.torch
        for h, pi in enumerate(self.plan.e3_column_halves()):
            self.derived[f"E3p{h}"] = e3.index_select(1, torch.as_tensor(pi, device=e3.device)).contiguous()
        for g, rho in enumerate(self.plan.e3_row_halves()):
            self.derived[f"E3r{g}"] = e3.index_select(0, torch.as_tensor(rho, device=e3.device)).contiguous()

    def _mat(self, key):
        if key in ("E1", "E2", "E3"):
            return self.mats[int(key[1]) - 1]
        return self.derived[key]

    def _buf(self, key):
        return getattr(self, key) if isinstance(key, str) else key  # a name or the tensor itself

    @classmethod
    def from_global(cls, u_host, cache, dev, group=None):
        import torch.distributed as tdist

        rank, P = tdist.get_rank(group), tdist.get_world_size(group)
        plan = SlabPlan(u_host.shape, P)
        local = dv.to_device(np.asfortranarray(plan.slab_a(u_host, rank)), np.complex128, dev)
        mats = cache.device_exps((np.complex128,) * 3, dev)
        return cls(plan, rank, dv.as_fortran(local).permute(2, 1, 0).reshape(-1), mats, NcclExchange(group))

    def _exec(self, prods, post=None):
        """Products through km_mumode_split; ``post`` (a km_pointop of the layout the last
        product writes) is fused into its epilogue when that product writes the plain layout
        along the last direction, else applied as an in-place pass over ``a`` afterwards."""
        stream = dv.stream_ptr(self.a.device)
        es = self.a.element_size()
        for idx, p in enumerate(prods):
            fuse = (post is not None and idx == len(prods) - 1 and p.plain_out()
                    and p.mu == len(self.plan.dims) - 1)
            mat = self._mat(p.mat)
            _native.check(self.lib.km_mumode_split(
                self._buf(p.src).data_ptr() + es * p.soff, self.code, mat.data_ptr(), self.mcodes[p.mu],
                self._buf(p.dst).data_ptr() + es * p.doff, p.m, p.nl, p.nmu, p.nr, p.kcb, p.kbs, p.ncb, p.nbs,
                p.acc, ctypes.byref(post) if fuse else None, stream))
            if fuse:
                post = None
        if post is not None:
            self._phase(self.a, post)

    def _run(self, calls, src, dst_final, scratch, post=None):
        """Serial products from (mu, m, nl, nmu, nr, kcb, kbs, ncb, nbs) tuples on explicit
        tensors (PeerSlabStepper's schedule)."""
        prods, cur = [], src
        for idx, (mu, m, nl, nmu, nr, kcb, kbs, ncb, nbs) in enumerate(calls):
            dst = dst_final if idx == len(calls) - 1 else scratch
            prods.append(Prod(mu, f"E{mu + 1}", m, nl, nmu, nr, kcb, kbs, ncb, nbs, cur, 0, dst, 0))
            cur = dst
        self._exec(prods, post)

    def _phase(self, buf, op):
        """In-place standalone pointwise pass over the local slab."""
        _native.check(self.lib.km_pointwise(buf.data_ptr(), buf.data_ptr(), self.code, self.plan.local,
                                            ctypes.byref(op), dv.stream_ptr(self.a.device)))

    def pre_exchange(self):
        before, _ = self.plan.even_calls() if self.layout == "A" else self.plan.odd_calls()
        self._run(before, self.a, self.send, self.w)
        return self.send

    def post_exchange(self):
        _, after = self.plan.even_calls() if self.layout == "A" else self.plan.odd_calls()
        self._run(after, self.recv, self.a, self.w)
        self.layout = "B" if self.layout == "A" else "A"

    def begin_step(self, **kw):
        """Everything of one step before and including the launch of its exchange(s): the
        products of each pre group, each followed by its all-to-all (asynchronous on the
        communicator's stream when ``comm`` is set; a virtual group moves the blocks itself).
        Returns the send buffer."""
        pre, _, size = self.plan.schedule(self.layout, self.overlap)
        self._works = []
        for h, group in enumerate(pre):
            self._exec(group)
            if self.comm is not None:
                self._works.append(self.comm.exchange_async(self.recv[h * size:(h + 1) * size],
                                                            self.send[h * size:(h + 1) * size]))
        return self.send

    def end_step(self, post=None, **kw):
        """The products after the exchange; post group h waits only for exchange h.  ``post``
        is a pointwise op on the layout the step ends in (fused where the kernel can)."""
        _, groups, _ = self.plan.schedule(self.layout, self.overlap)
        live = [i for i, g in enumerate(groups) if g]
        for h, group in enumerate(groups):
            if h < len(self._works):
                self._works[h].wait()
            if group:
                self._exec(group, post if h == live[-1] else None)
        self._works = []
        self.layout = "B" if self.layout == "A" else "A"

    def step(self, **kw):
        self.begin_step(**kw)
        self.end_step(**kw)

    def exchange_halves(self):
        """(number of exchanges, elements each) of a step from the current layout."""
        pre, _, size = self.plan.schedule(self.layout, self.overlap)
        return len(pre), size

    def local_state(self):
        """The local slab as a column-major (n1, n2, c3) [layout A] or (n1, c2, n3) [layout B] tensor view."""
        shape = self.plan.shape_a if self.layout == "A" else self.plan.shape_b
        return self.a.reshape(tuple(reversed(shape))).permute(2, 1, 0)

    def time_launches(self, reps=10):  # pragma: no cover - per-launch timing lives in LocalStepper
        return None


class SlabGpeStepper(SlabStepper):
    """Gross–Pitaevskii Strang steps (problems.py:548-565) of a 3D slab-decomposed state.

    Configuration 5 over P GPUs.  The nonlinear half-phase
    ``psi * exp(i coef (1 - |psi|^2 / w))`` is pointwise, so it runs on whichever
    layout the slab is in: its weight product ``w1[i1]*w2[i2]*w3[i3]`` is the
    global one seen through slab offsets (layout A: ``w3 + r*c3``; layout B:
    ``w2 + r*c2`` and the inner product ``(w1*w2)`` from row ``n1*r*c2``), so
    every element gets exactly the factors (and rounding) of the single-GPU step.
    As in :func:`problems.gpe_strang_run`, the closing half-phase of step k and
    the opening one of step k+1 are one ``repeat = 2`` rotation: fused into the
    direction-3 product's epilogue after even steps (that product writes layout
    B unblocked), a standalone in-place pass after odd steps (their last
    product writes layout A through the blocked input).  ``run(steps)`` (or
    ``begin_step(k=, steps=)`` / ``end_step(k=, steps=)`` around the exchange)
    applies the single opening and closing phases at the ends.
    """

    def __init__(self, plan, rank, local_a, mats, comm, weights_dev, inner_dev, half_tau, overlap=True):
        super().__init__(plan, rank, local_a, mats, comm, overlap=overlap)
        self.wdev = list(weights_dev)
        self.inner = inner_dev
        self.coef = 0.5 * half_tau  # problems.py:545
        self.launches_per_step += 1

    def _op(self, layout, repeat):
        n1, n2, n3 = self.plan.dims
        c2, c3, r = self.plan.c2, self.plan.c3, self.rank
        op = _native.PointOp()
        op.kind = _native.OP_GPE_PHASE
        op.d = 3
        op.repeat = repeat
        op.coef = self.coef
        w = [t.data_ptr() for t in self.wdev]
        if layout == "A":
            dims, w[2], inner = (n1, n2, c3), w[2] + 8 * r * c3, self.inner.data_ptr()
        else:
            dims, w[1], inner = (n1, c2, n3), w[1] + 8 * r * c2, self.inner.data_ptr() + 8 * n1 * r * c2
        for i in range(3):
            op.dims[i] = dims[i]
            op.weights[i] = w[i]
        op.inner_weights = inner
        return op

    def begin_step(self, k=0, steps=1, **kw):
        if k == 0:
            self._phase(self.a, self._op(self.layout, 1))
        return super().begin_step()

    def end_step(self, k=0, steps=1, **kw):
        out_layout = "B" if self.layout == "A" else "A"
        super().end_step(post=self._op(out_layout, 1 if k == steps - 1 else 2))

    def run(self, steps):
        for k in range(steps):
            self.step(k=k, steps=steps)

    @classmethod
    def from_global(cls, u_host, cache, weights, tau, dev, group=None):
        import torch.distributed as tdist

        from .tensor import inner_weight_product

        rank, P = tdist.get_rank(group), tdist.get_world_size(group)
        plan = SlabPlan(u_host.shape, P)
        local = dv.to_device(np.asfortranarray(plan.slab_a(u_host, rank)), np.complex128, dev)
        mats = cache.device_exps((np.complex128,) * 3, dev)
        w_dev = [dv.cached_vector(w, np.float64, dev) for w in weights]
        inner = dv.cached_vector(inner_weight_product(weights, u_host.shape), np.float64, dev)
        return cls(plan, rank, dv.as_fortran(local).permute(2, 1, 0).reshape(-1), mats, NcclExchange(group),
                   w_dev, inner, 0.5 * tau)


class SlabTdpotStepper(SlabStepper):
    """Configuration 4 over P GPUs: time-dependent-potential Strang steps of a slab state.

    The potential flows ``exp(-i x3 ∫ sin^2)`` over the two half steps are
    diagonal along direction 3 and commute with the other directions'
    products, so each rank folds them into its copy of E3 at the start of
    every step (``km_diag_phase_fold`` from the node vector and two scalars,
    as :func:`problems.tdpot_strang_step` does on one GPU) and the step is the
    plain slab step, one exchange per step.  ``begin_step(t=, tau=)``.
    """

    def __init__(self, plan, rank, local_a, mats, comm, x_nodes_dev, overlap=True):
        super().__init__(plan, rank, local_a, mats, comm, overlap=overlap)
        torch = dv.torch
        self.e3 = self.mats[2]
        self.folded = torch.empty_like(self.e3)
        self.x = x_nodes_dev
        # the derived forms of E3 (permuted columns, row halves) are folded per step from their
        # own unfolded copies, with the node vector permuted the same way
        self.base = {k: v.clone() for k, v in self.derived.items()}
        if self.overlap:
            self.x_cols = [self.x.index_select(0, torch.as_tensor(c, device=self.x.device))
                           for c in plan.e3_column_halves()]
            self.x_rows = [self.x.index_select(0, torch.as_tensor(r, device=self.x.device))
                           for r in plan.e3_row_halves()]
        self.launches_per_step += 1

    def _fold(self, src, dst, x_rows, x_cols, c_a, c_b):
        m, k = src.shape
        _native.check(self.lib.km_diag_phase_fold(src.data_ptr(), dst.data_ptr(), m, k, x_rows.data_ptr(),
                                                  x_cols.data_ptr(), c_a, c_b, dv.stream_ptr(self.a.device)))

    def begin_step(self, t=0.0, tau=0.0, **kw):
        from .problems import sin2_integral

        c_a, c_b = sin2_integral(t, t + 0.5 * tau), sin2_integral(t + 0.5 * tau, t + tau)
        if not self.overlap:
            self._fold(self.e3, self.folded, self.x, self.x, c_a, c_b)
            self.mats[2] = self.folded
        elif self.layout == "A":  # even step: the two column halves
            for h in range(2):
                self._fold(self.base[f"E3p{h}"], self.derived[f"E3p{h}"], self.x, self.x_cols[h], c_a, c_b)
        else:  # odd step: the two row halves
            for g in range(2):
                self._fold(self.base[f"E3r{g}"], self.derived[f"E3r{g}"], self.x_rows[g], self.x, c_a, c_b)
        return super().begin_step()

    def run(self, t0, tau, steps):
        for s_ in range(steps):
            self.step(t=t0 + s_ * tau, tau=tau)

    @classmethod
    def from_global(cls, u_host, cache, x_nodes, dev, group=None):
        import torch.distributed as tdist

        rank, P = tdist.get_rank(group), tdist.get_world_size(group)
        plan = SlabPlan(u_host.shape, P)
        local = dv.to_device(np.asfortranarray(plan.slab_a(u_host, rank)), np.complex128, dev)
        mats = cache.device_exps((np.complex128,) * 3, dev)
        x = dv.cached_vector(np.asarray(x_nodes, dtype=float), np.float64, dev)
        return cls(plan, rank, dv.as_fortran(local).permute(2, 1, 0).reshape(-1), mats, NcclExchange(group), x)


class PeerSlabStepper(SlabStepper):
    """:class:`SlabStepper` with the all-to-all fused into the products.

    The last product before each exchange stores its per-peer output blocks
    straight into the other ranks' receive buffers (``km_mumode_peer``: the
    epilogue's stores go over NVLink to symmetric-memory peer pointers), so
    the exchange overlaps the math tile by tile and no send buffer, pack pass
    or NCCL call is needed; a device-side barrier then orders the peers'
    writes before the local reads.  Receive buffers alternate between even and
    odd steps, so one barrier per step suffices: a rank writes a peer's buffer
    of parity p only after everybody passed the barrier of the step in
    between, i.e. after the peer has consumed it.
    """

    def __init__(self, plan, rank, local_a, mats, recv_pair, peer_ptrs, barrier):
        super().__init__(plan, rank, local_a, mats, comm=None, overlap=False)
        self.send = None
        self.recv_pair = recv_pair
        self.peer_ptrs = [(ctypes.c_void_p * plan.P)(*ptrs) for ptrs in peer_ptrs]
        self.barrier = barrier

    @classmethod
    def from_global(cls, u_host, cache, dev, group=None):
        import torch.distributed as tdist
        import torch.distributed._symmetric_memory as symm

        group = group or tdist.group.WORLD
        rank, P = tdist.get_rank(group), tdist.get_world_size(group)
        plan = SlabPlan(u_host.shape, P)
        local = dv.to_device(np.asfortranarray(plan.slab_a(u_host, rank)), np.complex128, dev)
        mats = cache.device_exps((np.complex128,) * 3, dev)
        if hasattr(symm, "enable_symm_mem_for_group"):
            symm.enable_symm_mem_for_group(group.group_name)
        bufs = [symm.empty(plan.local, dtype=dv.torch.complex128, device=dev) for _ in range(2)]
        handles = [symm.rendezvous(b, group) for b in bufs]
        ptrs = [list(h.buffer_ptrs) for h in handles]
        st = cls(plan, rank, dv.as_fortran(local).permute(2, 1, 0).reshape(-1), mats, tuple(bufs), ptrs,
                 lambda: handles[0].barrier(channel=0))
        st._handles = handles  # keep the mappings alive
        return st

    def pre_exchange(self):
        even = self.layout == "A"
        before, _ = self.plan.even_calls() if even else self.plan.odd_calls()
        self._run(before[:1], self.a, self.w, None)
        mu, m, nl, nmu, nr, kcb, kbs, ncb, nbs = before[1]
        # even: direction-2 rows in blocks of c2; odd: direction-1 fibers in blocks of c2*c3
        out_block, fiber_block = (ncb, 0) if even else (m, self.plan.c2 * self.plan.c3)
        _native.check(self.lib.km_mumode_peer(
            self.w.data_ptr(), self.code, self.mats[mu].data_ptr(), self.mcodes[mu], m, nl, nmu, nr, kcb, kbs,
            out_block, fiber_block, self.peer_ptrs[0 if even else 1], self.plan.P, self.rank * self.plan.block,
            dv.stream_ptr(self.a.device)))
        return None

    def post_exchange(self):
        even = self.layout == "A"
        _, after = self.plan.even_calls() if even else self.plan.odd_calls()
        self._run(after, self.recv_pair[0 if even else 1], self.a, self.w)
        self.layout = "B" if even else "A"

    def step(self):
        self.pre_exchange()
        self.barrier()
        self.post_exchange()


class NcclExchange:
    """Equal-split all-to-all of flat complex buffers over a torch.distributed group."""

    def __init__(self, group=None):
        import torch.distributed as tdist

        self.tdist = tdist
        self.group = group

    def exchange(self, recv, send):
        self.exchange_async(recv, send).wait()

    def exchange_async(self, recv, send):
        """Start the all-to-all; it runs on NCCL's stream after the work already queued on the
        current stream, and ``.wait()`` on the returned handle makes the current stream wait."""
        t = dv.torch
        r = t.view_as_real(recv) if recv.is_complex() else recv
        s = t.view_as_real(send) if send.is_complex() else send
        return self.tdist.all_to_all_single(r.reshape(-1), s.reshape(-1), group=self.group, async_op=True)


class VirtualSlabGroup:
    """P logical ranks of :class:`SlabStepper` in ONE process on ONE device.

    The exchange is a local block permutation (recv_r[block s] = send_s[block r]),
    so the split-layout kernels and the step schedule run exactly as on P GPUs
    while nothing waits on another process (SURVEY §4 "virtual-rank" test).
    """

    def __init__(self, u_host, cache, dev, P, exchange="nccl", kind="plain", weights=None, tau=None,
                 x_nodes=None, overlap=True):
        """``kind``: "plain" (exact steps), "gpe" (SlabGpeStepper: ``weights``, ``tau``) or
        "tdpot" (SlabTdpotStepper: ``x_nodes``)."""
        self.plan = SlabPlan(u_host.shape, P)
        self.exchange = exchange
        mats = cache.device_exps((np.complex128,) * 3, dev)
        self.ranks = []
        locals_ = []
        for r in range(P):
            local = dv.to_device(np.asfortranarray(self.plan.slab_a(u_host, r)), np.complex128, dev)
            locals_.append(local.permute(2, 1, 0).reshape(-1))
        if exchange == "peer":
            if kind != "plain":
                raise ValueError("the peer exchange steps plain propagators only")
            recv = [(dv.torch.empty_like(x), dv.torch.empty_like(x)) for x in locals_]
            ptrs = [[recv[s][k].data_ptr() for s in range(P)] for k in range(2)]
            for r in range(P):
                self.ranks.append(PeerSlabStepper(self.plan, r, locals_[r], mats, recv[r], ptrs, lambda: None))
        elif kind == "gpe":
            from .tensor import inner_weight_product

            w_dev = [dv.cached_vector(w, np.float64, dev) for w in weights]
            inner = dv.cached_vector(inner_weight_product(weights, u_host.shape), np.float64, dev)
            for r in range(P):
                self.ranks.append(SlabGpeStepper(self.plan, r, locals_[r], list(mats), None, w_dev, inner,
                                                 0.5 * tau, overlap=overlap))
        elif kind == "tdpot":
            x = dv.cached_vector(np.asarray(x_nodes, dtype=float), np.float64, dev)
            for r in range(P):
                self.ranks.append(SlabTdpotStepper(self.plan, r, locals_[r], list(mats), None, x, overlap=overlap))
        else:
            for r in range(P):
                self.ranks.append(SlabStepper(self.plan, r, locals_[r], mats, comm=None, overlap=overlap))

    def step(self, **kw):
        if self.exchange == "peer":
            for st in self.ranks:  # every rank stores its blocks into the others' receive buffers
                st.pre_exchange()
            for st in self.ranks:
                st.post_exchange()
            return
        P = self.plan.P
        halves, size = self.ranks[0].exchange_halves()
        blk = size // P
        sends = [st.begin_step(**kw) for st in self.ranks]
        for h in range(halves):  # the all-to-all of each half: recv_r[h][s] = send_s[h][r]
            base = h * size
            for r, st in enumerate(self.ranks):
                for s in range(P):
                    st.recv[base + s * blk:base + (s + 1) * blk].copy_(sends[s][base + r * blk:base + (r + 1) * blk])
        for st in self.ranks:
            st.end_step(**kw)

    def gather(self):
        """The global state as a host numpy array (column-major)."""
        n1, n2, n3 = self.plan.dims
        out = np.empty((n1, n2, n3), dtype=np.complex128, order="F")
        for r, st in enumerate(self.ranks):
            loc = dv.to_host(st.local_state())
            if st.layout == "A":
                out[:, :, r * self.plan.c3:(r + 1) * self.plan.c3] = loc
            else:
                out[:, r * self.plan.c2:(r + 1) * self.plan.c2, :] = loc
        return out
