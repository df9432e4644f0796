"""Config 2 eager step (pipe flow 1024^2 f64) under the CUDA activity profiler: per-kernel
device durations and the gaps between them, with and without the stream-K cut, next to the
same two products launched directly through km_mumode (tools/ab_probe.py's view).

    python tools/pipe_trace.py
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2103_01691_b200 as km  # noqa: E402
from paper_2103_01691_b200 import _device as dv, _native  # noqa: E402

DEV = torch.device("cuda", 0)
n = 1024
cache = km.prepare(km.pipeflow_factors(n), 4.0 / 16)
rho, z = km.fd.pipeflow_grids(n)
c0 = np.asfortranarray(np.exp(-8.0 * (rho.points - 2.55) ** 2)[:, None] * np.exp(-8.0 * (z.points - 1.5) ** 2)[None, :])
t = dv.to_device(c0, np.float64, DEV)


def trace(fn, reps=6):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
    ev = sorted((e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA),
                key=lambda e: e.time_range.start)
    last = None
    for e in ev[-6:]:
        gap = (e.time_range.start - last) if last is not None else 0.0
        print(f"    {e.name[:60]:60s} {e.time_range.elapsed_us():7.1f} us  gap {gap:6.1f} us")
        last = e.time_range.end
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        fn()
    e1.record()
    e1.synchronize()
    print(f"  events: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us per call")


lib = _native.lib()
e1d, e2d = cache.device_exps((np.float64, np.float64), DEV)
mid = torch.empty(n * n, dtype=torch.float64, device=DEV)
out = torch.empty(n * n, dtype=torch.float64, device=DEV)


def direct():
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    _native.check(lib.km_mumode(ctypes.c_void_p(t.data_ptr()), 1, ctypes.c_void_p(e1d.data_ptr()), 1,
                                ctypes.c_void_p(mid.data_ptr()), n, 1, n, n, None, s))
    _native.check(lib.km_mumode(ctypes.c_void_p(mid.data_ptr()), 1, ctypes.c_void_p(e2d.data_ptr()), 1,
                                ctypes.c_void_p(out.data_ptr()), n, n, n, 1, None, s))


for name, pol in (("stream-K", _native.POLICY_AUTO), ("whole tiles", _native.POLICY_NO_STREAMK)):
    _native.check(lib.km_set_kernel_policy(pol))
    print(name, "km.step:")
    trace(lambda: km.step(cache, t))
    print(name, "two km_mumode calls:")
    dv._bind_stream_workspace(0, torch.cuda.current_stream().cuda_stream)
    trace(direct)
_native.check(lib.km_set_kernel_policy(_native.POLICY_AUTO))
