"""One long-contraction complex64 product (direction 1 of n x n x 64, K' = 2n): the HALVES kernel up to
K' = 1024, the chunked tcgen05 kernel beyond (or under KM_POLICY_NO_TC_HALVES)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2103_01691_b200 as km  # noqa: E402
from paper_2103_01691_b200 import _device as dv  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
mu = int(sys.argv[2]) if len(sys.argv) > 2 else 1
rng = np.random.default_rng(0)
shape = (n, n, 64)
u = dv.to_device(np.asfortranarray((rng.standard_normal(shape) + 1j * rng.standard_normal(shape)).astype(np.complex64)),
                 np.complex64, torch.device("cuda", 0))
m = shape[mu - 1]
mat = ((rng.standard_normal((m, m)) + 1j * rng.standard_normal((m, m))) / np.sqrt(m)).astype(np.complex64)
km.mu_mode_product(u, mat, mu)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    km.mu_mode_product(u, mat, mu)
e1.record()
e1.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"n={n} mu={mu}: {ms:.3f} ms, {8 * n * n * 64 * m / ms / 1e9:.1f} TFLOP/s complex")
