"""Steppers that keep the state resident on the device(s) across steps.

* :class:`LocalStepper` — one GPU.  The exact step ``u x_1 E_1 ... x_d E_d``
  runs as one ``km_tucker`` call per step over three device buffers (state,
  one scratch, next state): the reference's acceptance criterion 9 bound of
  3x the state (test_acceptance.py:298-321) holds on the device.
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
        self.launches_per_step = self.d + (1 if pre is not None else 0)
        self.lib = _native.lib()

    def step(self):
        """``a <- a x_1 E_1 ... x_d E_d``; the input buffer doubles as the second scratch."""
        stream = dv.stream_ptr(self.a.device)
        _native.check(self.lib.km_tucker(
            self.a.data_ptr(), self.code, self.d, self._c_dims, self._c_mats, self._c_codes, self._c_rows,
            self.b.data_ptr(), self.w.data_ptr(), self.a.data_ptr(),
            None if self.pre is None else ctypes.byref(self.pre),
            None if self.post is None else ctypes.byref(self.post), stream))
        self.a, self.b = self.b, self.a

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


class SlabStepper:
    """Exact steps of a 3D state split into slabs across the ranks of a process group.

    Placeholder until the fused all-to-all path lands; see DESIGN.md §Multi-GPU.
    """

    launches_per_step = 3

    @classmethod
    def from_global(cls, u_host, cache, dev):  # pragma: no cover - filled in with the NCCL path
        raise NotImplementedError("multi-GPU slab stepping is not built yet")


del np
