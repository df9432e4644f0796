"""A/B of the drop-in pipeline's plan knobs (_pipeline.FIB_PIECES, TAIL_SHIFTS): e2e steps/s of
step(cache, pinned numpy 256^3 c128), 20 calls per setting, settings interleaved twice."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2103_01691_b200 as km  # noqa: E402
from paper_2103_01691_b200 import _pipeline  # noqa: E402

u, cache = bench.build_inputs()
N = u.shape[0]
pinned = torch.empty((N, N, N), dtype=torch.complex128, pin_memory=True)
pinned.numpy()[...] = u.transpose(2, 1, 0)
host = pinned.numpy().transpose(2, 1, 0)
settings = [(4, (3, 4, 5, 6)), (8, (3, 4, 5, 6)), (8, (3, 4, 5, 6, 7)), (4, (3, 4, 5, 6, 7))]
for rep in range(2):
    for pieces, tail in settings:
        _pipeline.FIB_PIECES, _pipeline.TAIL_SHIFTS = pieces, tail
        for _ in range(3):
            km.step(cache, host)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(20):
            out = km.step(cache, host)
        torch.cuda.synchronize()
        print(f"pieces={pieces} tail={tail}: {20 / (time.perf_counter() - t0):.2f} steps/s")
