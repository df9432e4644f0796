"""Configuration 1 through the public API: ``for _ in range(10): u = km.step(cache, u)`` on a
device tensor (host launch path included), against the device-only CUDA-graph run.

    python tools/api_loop_probe.py
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2103_01691_b200 as km  # noqa: E402
from paper_2103_01691_b200 import _device as dv  # noqa: E402

dev = torch.device("cuda", 0)
for n in (16, 32, 64):
    rng = np.random.default_rng(0)
    u0 = dv.to_device(np.asfortranarray(rng.standard_normal((n,) * 3) + 1j * rng.standard_normal((n,) * 3)),
                      np.complex128, dev)
    d2 = km.heat_factors(n, 2).factors[0]
    cache = km.prepare(km.KroneckerOp((1j * d2,) * 3), 0.01)

    def ten():
        u = u0
        for _ in range(10):
            u = km.step(cache, u)
        return u

    for _ in range(20):
        ten()
    torch.cuda.synchronize()
    reps = 200
    t0 = time.perf_counter()
    for _ in range(reps):
        ten()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / reps
    print(f"n={n}: 10 x km.step(cache, device tensor) {wall * 1e6:.1f} us wall ({wall * 1e5:.1f} us per step)", flush=True)
