"""complex64 exact steps on tcgen05 at 256^3 and 512^3 (512: direction 1, K' = 1024, runs two folded accumulation chains),
device time per step and parity against the complex128 and complex64 oracle steps."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2103_01691_b200 as km  # noqa: E402
from oracle import kronmode_oracle as orc  # noqa: E402
from paper_2103_01691_b200 import _device as dv, _native  # noqa: E402

DEV = torch.device("cuda", 0)
for n in (256, 512):
    rng = np.random.default_rng(0)
    u = np.asfortranarray((rng.standard_normal((n,) * 3) + 1j * rng.standard_normal((n,) * 3)).astype(np.complex64))
    d2 = km.heat_factors(n, 2).factors[0]
    c128 = km.prepare(km.KroneckerOp((1j * d2,) * 3), 0.01)
    c64 = km.PropagatorCache(0.01, tuple(e.astype(np.complex64) for e in c128.exps))
    t = dv.to_device(u, np.complex64, DEV)
    res = {}
    for name, pol in (("tcgen05", _native.POLICY_AUTO), ("dmma", _native.POLICY_NO_TMA)):
        _native.check(_native.lib().km_set_kernel_policy(pol))
        km.step(c64, t)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            out = km.step(c64, t)
        e1.record()
        e1.synchronize()
        res[name] = (e0.elapsed_time(e1) / 5, dv.to_host(out).copy())
    _native.check(_native.lib().km_set_kernel_policy(_native.POLICY_AUTO))
    want128 = orc.step(c128.exps, u.astype(np.complex128))
    want64 = orc.step(c64.exps, u)
    for name, (ms, got) in res.items():
        print(f"n={n} {name}: {ms:.3f} ms/step, {8 * 3 * n**4 / ms / 1e9:.1f} TFLOP/s, "
              f"rel_l2 vs c128 {orc.rel_l2(got, want128):.2e}, vs ref c64 {orc.rel_l2(got, want64):.2e}")
