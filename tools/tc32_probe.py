"""Time complex64 products: tcgen05 3xTF32 kernel vs the DMMA path (n=256^3)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2103_01691_b200 as km  # noqa: E402
from paper_2103_01691_b200 import _device as dv, _native  # noqa: E402

n = 256
dev = torch.device("cuda", 0)
rng = np.random.default_rng(0)
u = np.asfortranarray((rng.standard_normal((n,) * 3) + 1j * rng.standard_normal((n,) * 3)).astype(np.complex64))
d2 = km.heat_factors(n, 2).factors[0]
c128 = km.prepare(km.KroneckerOp((1j * d2,) * 3), 0.01)
cache = km.PropagatorCache(0.01, tuple(e.astype(np.complex64) for e in c128.exps))
t = dv.to_device(u, np.complex64, dev)


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


lib = _native.lib()
for mu in (1, 2, 3):
    ms = timeit(lambda: km.mu_mode_product(t, cache.exps[mu - 1], mu))
    lib.km_set_kernel_policy(1)
    ms2 = timeit(lambda: km.mu_mode_product(t, cache.exps[mu - 1], mu))
    lib.km_set_kernel_policy(0)
    print(f"c64 mode {mu}: tcgen05 {ms:.3f} ms ({8 * n**4 / ms / 1e9:.1f} TFLOP/s)   dmma {ms2:.3f} ms")
ms = timeit(lambda: km.step(cache, t))
print(f"c64 step: {ms:.3f} ms = {1e3 / ms:.1f} steps/s ({8 * 3 * n**4 / ms / 1e9:.1f} TFLOP/s)")
