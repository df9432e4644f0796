"""complex64 exact step time on tcgen05 (CUDA events, 20 steps after warm-up) at n^3.

    python tools/c64_step_time.py [n ...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2103_01691_b200 as km  # noqa: E402

dev = torch.device("cuda", 0)
for n in [int(a) for a in sys.argv[1:]] or [256, 512]:
    g = torch.Generator(device=dev).manual_seed(0)
    u = torch.randn((n, n, n), dtype=torch.complex64, device=dev, generator=g).permute(2, 1, 0)
    d2 = km.heat_factors(n, 2).factors[0]
    c128 = km.prepare(km.KroneckerOp((1j * d2,) * 3), 0.01)
    cache = km.PropagatorCache(0.01, tuple(e.astype(np.complex64) for e in c128.exps))
    for _ in range(3):
        km.step(cache, u)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        km.step(cache, u)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"n={n}: c64 step {ms:.4f} ms, {8 * 3 * n**4 / ms / 1e9:.1f} TFLOP/s complex")
