"""Break down the host-pipelined drop-in step (numpy in pinned memory -> numpy)."""
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


def timeit(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        r = fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3, r


for parts in (16, 8, 4, 8, 16, 32):
    from paper_2103_01691_b200 import _pipeline as pl
    orig = pl.tucker_host_pipelined

    def patched(*a, **k):
        k["parts"] = parts
        return orig(*a, **k)

    pl.tucker_host_pipelined = patched
    ms, _ = timeit(lambda: km.step(cache, host))
    pl.tucker_host_pipelined = orig
    print(f"step host pipelined parts={parts}: {ms:.2f} ms")
ms, _ = timeit(lambda: torch.empty((N, N, N), dtype=torch.complex128, pin_memory=True))
print(f"pinned alloc: {ms:.3f} ms")
d = torch.empty((N, N, N), dtype=torch.complex128, device="cuda")
ms, _ = timeit(lambda: d.copy_(pinned, non_blocking=True))
print(f"H2D 268MB: {ms:.2f} ms")
ms, _ = timeit(lambda: pinned.copy_(d, non_blocking=True))
print(f"D2H 268MB: {ms:.2f} ms")
t = torch.from_numpy(host.reshape(-1, order="F"))
ms, _ = timeit(lambda: t.is_pinned())
print(f"is_pinned: {ms:.3f} ms")
