"""Per-rank compute of the slab decomposition (256^3 c128), measured on one GPU.

Each rank of a P-GPU run executes exactly rank 0's products here (same shapes,
same blocked layouts); the exchange is left out.  Prints the per-rank time per
step and its fraction of the DMMA roofline for the rank's share of the work.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2103_01691_b200 as km  # noqa: E402
from paper_2103_01691_b200 import dist  # noqa: E402

DEV = torch.device("cuda", 0)
PEAK = 37.14e12
n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
rng = np.random.default_rng(0)
u = np.asfortranarray(rng.standard_normal((n,) * 3) + 1j * rng.standard_normal((n,) * 3))
d2 = km.heat_factors(n, 2).factors[0]
cache = km.prepare(km.KroneckerOp((1j * d2,) * 3), 0.01)
flop = 8 * 3 * n**4
for P in (1, 2, 4, 8):
    for exch in ("nccl", "peer"):
        g = dist.VirtualSlabGroup(u, cache, DEV, P, exchange=exch)
        r0 = g.ranks[0]

        def one():
            r0.pre_exchange()
            r0.post_exchange()

        for _ in range(4):
            one()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 20
        e0.record()
        for _ in range(reps):
            one()
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / reps
        print(f"P={P} {exch}: rank-0 products {ms:.3f} ms/step -> {flop / P / (ms * 1e-3) / PEAK:.3f} of DMMA peak")
        del g
        torch.cuda.empty_cache()
