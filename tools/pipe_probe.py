"""Config 2 (pipe flow 1024^2 f64, one exact step): device time per step with
and without the stream-K cut, and parity against the oracle.

    python tools/pipe_probe.py [n]
"""
import gc
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2103_01691_b200 as km  # noqa: E402
from oracle import kronmode_oracle as orc  # noqa: E402
from paper_2103_01691_b200 import _device as dv, _native  # noqa: E402

DEV = torch.device("cuda", 0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
cache = km.prepare(km.pipeflow_factors(n), 4.0 / 16)
rho, z = km.fd.pipeflow_grids(n)
c0 = np.asfortranarray(np.exp(-8.0 * (rho.points - 2.55) ** 2)[:, None] * np.exp(-8.0 * (z.points - 1.5) ** 2)[None, :])
want = orc.step(cache.exps, c0)
# ~0.5 s of products first: the first run of a fresh process otherwise times the clock ramp
t0 = dv.to_device(c0, c0.dtype, DEV)
for _ in range(3000):
    km.step(cache, t0)
torch.cuda.synchronize()
for cplx in (False, True):
    u = c0 * (1 + 1j) if cplx else c0
    t = dv.to_device(u, u.dtype, DEV)
    for name, pol in (("stream-K", _native.POLICY_AUTO), ("whole tiles", _native.POLICY_NO_STREAMK)):
        _native.check(_native.lib().km_set_kernel_policy(pol))
        for _ in range(3):
            km.step(cache, t)
        torch.cuda.synchronize()
        gc.collect()  # a collector pause inside the timed loop idles the GPU between launches
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50):
            out = km.step(cache, t)
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / 50
        got = dv.to_host(out)
        ref = want * (1 + 1j) if cplx else want
        flop = (4 if cplx else 2) * 2 * n ** 3
        print(f"n={n} {'c128' if cplx else 'f64'} {name}: {ms * 1e3:.1f} us/step, {flop / ms / 1e9:.1f} TFLOP/s, "
              f"rel_l2 {orc.rel_l2(got, ref):.2e}")
_native.check(_native.lib().km_set_kernel_policy(_native.POLICY_AUTO))
