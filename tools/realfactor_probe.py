"""Real factor x complex128 tensor products (the Hermite transforms of config 3) at 256^3:
device time per direction, TFLOP/s at 4 flop per complex x real multiply-add, fraction of the
measured DMMA peak.  python tools/realfactor_probe.py [n]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2103_01691_b200 as km  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
u = torch.randn((n, n, n), dtype=torch.complex128, device=dev, generator=g).permute(2, 1, 0)
mat = torch.from_numpy(np.random.default_rng(0).standard_normal((n, n))).to(dev)
for mu in (1, 2, 3):
    km.mu_mode_product(u, mat, mu)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        km.mu_mode_product(u, mat, mu)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 10
    tf = 4 * n**4 / ms / 1e9
    print(f"n={n} mu={mu}: {ms:.3f} ms, {tf:.1f} TFLOP/s, {tf / 37.14:.3f} of DMMA peak")
