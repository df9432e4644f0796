"""Parity of the tcgen05 complex64 products against the complex128 oracle (prints rel. l2 per direction)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2103_01691_b200 as km  # noqa: E402
from oracle import kronmode_oracle as orc  # noqa: E402

rng = np.random.default_rng(0)
shape = (256, 256, 128)
u = np.asfortranarray((rng.standard_normal(shape) + 1j * rng.standard_normal(shape)).astype(np.complex64))
for mu in (1, 2, 3):
    n = shape[mu - 1]
    mat = ((rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / np.sqrt(n)).astype(np.complex64)
    got = km.mu_mode_product(u, mat, mu)
    want64 = orc.mu_mode_product(u, mat, mu)
    want128 = orc.mu_mode_product(u.astype(np.complex128), mat.astype(np.complex128), mu)
    print(f"mu={mu}: vs c128 {orc.rel_l2(got, want128):.2e}   reference c64 vs c128 {orc.rel_l2(want64, want128):.2e}")
