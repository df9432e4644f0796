"""cProfile of the public API's host path on a small device tensor (where the Python layer
is the critical path): km.step(cache, tensor) and mu_mode_product(tensor, numpy matrix).

    python tools/host_profile.py [calls]
"""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2103_01691_b200 as km  # noqa: E402
from paper_2103_01691_b200 import _device as dv  # noqa: E402

calls = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
dev = torch.device("cuda", 0)
n = 16
rng = np.random.default_rng(0)
u = dv.to_device(np.asfortranarray(rng.standard_normal((n,) * 3) + 1j * rng.standard_normal((n,) * 3)),
                 np.complex128, dev)
mat = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / n
cache = km.PropagatorCache(0.1, (mat, mat, mat))
for name, fn in (("step", lambda: km.step(cache, u)), ("mu_mode_product", lambda: km.mu_mode_product(u, mat, 2))):
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(calls):
        fn()
    torch.cuda.synchronize()
    print(f"{name}: {(time.perf_counter() - t0) / calls * 1e6:.1f} us per call", flush=True)
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(calls):
        fn()
    pr.disable()
    torch.cuda.synchronize()
    pstats.Stats(pr).sort_stats("tottime").print_stats(18)
