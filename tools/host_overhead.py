"""Host-side cost per call of the public API on small device tensors (wall
clock, device work negligible): where the Python layer sits on the critical
path of launch-bound loops (Krylov matvecs, small states).

    python tools/host_overhead.py
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
n = 16
rng = np.random.default_rng(0)
for dt in (np.complex128, np.complex64):
    u = dv.to_device(np.asfortranarray((rng.standard_normal((n,) * 3) + 1j * rng.standard_normal((n,) * 3)).astype(dt)),
                     dt, dev)
    mat = ((rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / n).astype(dt)
    mat_dev = dv.to_device(np.ascontiguousarray(mat), dt, dev)
    cache = km.PropagatorCache(0.1, (mat, mat, mat))
    cases = {
        "mu_mode_product(tensor, numpy mat)": lambda: km.mu_mode_product(u, mat, 2),
        "mu_mode_product(tensor, device mat)": lambda: km.mu_mode_product(u, mat_dev, 2),
        "step(cache, tensor)": lambda: km.step(cache, u),
        "tucker(tensor, [numpy]*3)": lambda: km.tucker(u, [mat, mat, mat]),
    }
    for name, fn in cases.items():
        for _ in range(20):
            fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(200):
            fn()
        torch.cuda.synchronize()
        us = (time.perf_counter() - t0) / 200 * 1e6
        print(f"{np.dtype(dt).name:10s} {name:40s} {us:8.1f} us/call")
