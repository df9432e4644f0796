"""float32 x float32 steps: the fiber-pair tcgen05 route against the DMMA route (policy
NO_TMA sends every product to the cp.async DMMA kernel) and the float64 result.

    python tools/f32_probe.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2103_01691_b200 as km  # noqa: E402
from oracle import kronmode_oracle as orc  # noqa: E402
from paper_2103_01691_b200 import _device as dv, tensor  # noqa: E402

DEV = torch.device("cuda", 0)
for n in (128, 256):
    rng = np.random.default_rng(n)
    u = np.asfortranarray(rng.standard_normal((n,) * 3).astype(np.float32))
    d2 = km.heat_factors(n, 2).factors[0]
    cache = km.prepare(km.KroneckerOp((d2,) * 3), 1e-4)
    mats = [e.astype(np.float32) for e in cache.exps]
    t = dv.to_device(u, np.float32, DEV)
    want = orc.tucker(u.astype(np.float64), [m.astype(np.float64) for m in mats])
    for name, rr32 in (("fiber pairs on tcgen05", True), ("DMMA (widened)", False)):
        tensor._RR32_ON_TC = rr32

        def fn():
            return km.tucker(t, mats)

        for _ in range(3):
            r = fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            r = fn()
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / 20
        print(f"n={n} {name}: {ms * 1e3:.1f} us/step, {2 * 3 * n ** 4 / ms / 1e9:.1f} TFLOP/s (real), "
              f"rel_l2 vs float64 {orc.rel_l2(dv.to_host(r), want):.2e}", flush=True)
tensor._RR32_ON_TC = True
