"""Device timeline of one drop-in step(cache, numpy) call (host-pipelined path):
H2D slabs, per-slab products, direction-d row blocks and D2H blocks, in ms
from the call's first event.  python tools/e2e_timeline.py [--pageable]
(--pageable: an ordinary numpy input, staged through the page-locked ring)"""
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
if "--pageable" in sys.argv:
    import numpy as np

    host = np.asfortranarray(u.copy())
for _ in range(3):
    km.step(cache, host)
torch.cuda.synchronize()
_pipeline._trace_on = True
t0 = time.perf_counter()
km.step(cache, host)
t1 = time.perf_counter()
wall = (t1 - t0) * 1e3
torch.cuda.synchronize()
first = _pipeline.TRACE[0][1]
print("  device   host-issue  event   (ms from the first event; host-issue from the call)")
for label, ev, th in _pipeline.TRACE:
    print(f"{first.elapsed_time(ev):8.3f}  {1e3 * (th - t0):8.3f}  {label}")
print(f"wall {wall:.3f} ms; host time before the first event {1e3 * (_pipeline.TRACE[0][2] - t0):.3f} ms")
