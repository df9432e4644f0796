"""complex64 steps on tcgen05: device time and error against the complex128 result and against
the reference's own complex64 arithmetic, for comparing accumulation-chain settings between
library builds (KMB200_LIB).

    python tools/c64_chain_probe.py [n ...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2103_01691_b200 as km  # noqa: E402
from oracle import kronmode_oracle as orc  # noqa: E402
from paper_2103_01691_b200 import _device as dv  # noqa: E402

DEV = torch.device("cuda", 0)
for n in [int(a) for a in sys.argv[1:]] or [256, 512]:
    rng = np.random.default_rng(n)
    u = np.asfortranarray((rng.standard_normal((n,) * 3) + 1j * rng.standard_normal((n,) * 3)).astype(np.complex64))
    d2 = km.heat_factors(n, 2).factors[0]
    cache = km.prepare(km.KroneckerOp((1j * d2,) * 3), 0.01)
    e64 = [e.astype(np.complex64) for e in cache.exps]
    t = dv.to_device(u, np.complex64, DEV)
    mats = [dv.matrix_to_device(e, np.complex64, DEV) for e in e64]
    for _ in range(3):
        r = km.tucker(t, mats)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        r = km.tucker(t, mats)
    e1.record()
    e1.synchronize()
    got = dv.to_host(r).astype(np.complex128)
    ref64 = orc.tucker(u, e64)  # the reference's complex64 arithmetic
    ref128 = orc.tucker(u.astype(np.complex128), [e.astype(np.complex128) for e in e64])
    print(f"n={n}: {e0.elapsed_time(e1) / 10:.3f} ms/step; rel l2 vs complex128 {orc.rel_l2(got, ref128):.2e}, "
          f"vs reference complex64 {orc.rel_l2(got, ref64.astype(np.complex128)):.2e} "
          f"(reference complex64 vs complex128 {orc.rel_l2(ref64.astype(np.complex128), ref128):.2e})", flush=True)
