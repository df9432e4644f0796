"""Short workload for ncu: complex64 256^3 exact steps (tcgen05 kernels)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2103_01691_b200 as km  # noqa: E402
from paper_2103_01691_b200 import _device as dv  # noqa: E402

n = 256
rng = np.random.default_rng(0)
u = np.asfortranarray((rng.standard_normal((n,) * 3) + 1j * rng.standard_normal((n,) * 3)).astype(np.complex64))
d2 = km.heat_factors(n, 2).factors[0]
c128 = km.prepare(km.KroneckerOp((1j * d2,) * 3), 0.01)
cache = km.PropagatorCache(0.01, tuple(e.astype(np.complex64) for e in c128.exps))
t = dv.to_device(u, np.complex64, torch.device("cuda", 0))
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    t = km.step(cache, t)
torch.cuda.synchronize()
print("ok")
