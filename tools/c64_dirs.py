"""complex64 512^3 (or n^3) products per direction on tcgen05: device time and
tensor-core rate (8 flop per complex multiply-add).  Direction 1 at n = 512
(K' = 1024) runs the chunked kernel.

    python tools/c64_dirs.py [n]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2103_01691_b200 as km  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
u = torch.randn((n, n, n), dtype=torch.complex64, device=dev, generator=g).permute(2, 1, 0)  # column-major
rng = np.random.default_rng(0)
mat = ((rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / np.sqrt(n)).astype(np.complex64)
from paper_2103_01691_b200 import _native  # noqa: E402

for mu, pol in ((1, _native.POLICY_AUTO), (1, _native.POLICY_NO_TC_HALVES), (2, 0), (3, 0)):
    _native.check(_native.lib().km_set_kernel_policy(pol))
    km.mu_mode_product(u, mat, mu)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        km.mu_mode_product(u, mat, mu)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 5
    tag = " (no halves: chunked)" if pol else ""
    print(f"n={n} mu={mu}{tag}: {ms:.3f} ms, {8 * n**4 / ms / 1e9:.1f} TFLOP/s complex")
_native.check(_native.lib().km_set_kernel_policy(_native.POLICY_AUTO))
