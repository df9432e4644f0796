"""Host memcpy bandwidth into page-locked memory with 1..16 threads (the pageable-input
staging of the drop-in path, _pipeline._parallel_copy).

    python tools/host_copy_bw.py
"""
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

n = 32 << 20  # 32 MB blocks, as the staging ring
src = np.random.default_rng(0).standard_normal(256 << 20 >> 3)  # 256 MB pageable
dst = torch.empty(256 << 20, dtype=torch.uint8, pin_memory=True).numpy().view(np.float64)
for threads in (1, 2, 4, 8, 12, 16):
    pool = ThreadPoolExecutor(max_workers=threads)
    cuts = [src.size * i // threads for i in range(threads + 1)]

    def run():
        list(pool.map(lambda i: np.copyto(dst[cuts[i]:cuts[i + 1]], src[cuts[i]:cuts[i + 1]]), range(threads)))

    run()
    t0 = time.perf_counter()
    for _ in range(5):
        run()
    el = (time.perf_counter() - t0) / 5
    print(f"{threads:2d} threads: {src.nbytes / el / 1e9:.1f} GB/s", flush=True)
    pool.shutdown()
