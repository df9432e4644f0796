"""Per-call timeline of the drop-in host step to expose warm-up effects."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2103_01691_b200 as km  # noqa: E402

u, cache = bench.build_inputs()
N = u.shape[0]
pinned = torch.empty((N, N, N), dtype=torch.complex128, pin_memory=True)
pinned.numpy()[...] = u.transpose(2, 1, 0)
host = pinned.numpy().transpose(2, 1, 0)
d = torch.empty((N, N, N), dtype=torch.complex128, device="cuda")
ts = []
t00 = time.perf_counter()
for i in range(40):
    t0 = time.perf_counter()
    out = km.step(cache, host)
    ts.append((time.perf_counter() - t0) * 1e3)
print("per-call ms:", " ".join(f"{t:.1f}" for t in ts))
ts = []
for i in range(20):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    d.copy_(pinned, non_blocking=True)
    torch.cuda.synchronize()
    ts.append((time.perf_counter() - t0) * 1e3)
print("H2D ms:", " ".join(f"{t:.2f}" for t in ts))
