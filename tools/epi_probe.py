"""Cost of the fused GPE phase epilogue: the direction-3 product alone, with the
phase fused (repeat 1 and 2), and the standalone pointwise pass, at n^3 c128.

    python tools/epi_probe.py [n] [once]
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2103_01691_b200 as km  # noqa: E402
from oracle import kronmode_oracle as orc  # noqa: E402
from paper_2103_01691_b200 import _device as dv, _native  # noqa: E402
from paper_2103_01691_b200.problems import _gpe_op, _inner_weight_product, weighted_vortex_state  # noqa: E402
from paper_2103_01691_b200.tensor import run_tucker  # noqa: E402

dev = torch.device("cuda", 0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 256


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


grids, lin_op, weights = km.gpe_setup(n)
psi = weighted_vortex_state(grids, weights)
cache = km.prepare(lin_op, 0.1)
p = dv.to_device(psi, np.complex128, dev)
w_dev = [dv.cached_vector(w, np.float64, dev) for w in weights]
inner = dv.cached_vector(_inner_weight_product(weights, psi.shape), np.float64, dev)
keep = w_dev + [inner]
mats = [None, None, cache.exps[2]]
ops = {r: _gpe_op(psi.shape, w_dev, 0.05, inner, r) for r in (1, 2)}
if len(sys.argv) > 2 and sys.argv[2] == "once":  # one fused launch, for ncu
    run_tucker(p, mats, post=ops[2], keepalive=keep)
    torch.cuda.synchronize()
    sys.exit(0)
t_plain = timeit(lambda: run_tucker(p, mats))
t_r1 = timeit(lambda: run_tucker(p, mats, post=ops[1], keepalive=keep))
t_r2 = timeit(lambda: run_tucker(p, mats, post=ops[2], keepalive=keep))
out = torch.empty_like(p)
lib = _native.lib()
t_pw = timeit(lambda: lib.km_pointwise(p.data_ptr(), out.data_ptr(), _native.KM_C128, p.numel(),
                                       ctypes.byref(ops[1]), dv.stream_ptr(dev)))
# parity of the fused epilogue against the oracle's phase (problems.py:542-545)
got = dv.to_host(run_tucker(p, mats, post=ops[2], keepalive=keep))
want = orc.mu_mode_product(psi, cache.exps[2], 3)
wp = np.ones(psi.shape, order="F")
for ax, w in enumerate(weights):
    wp = wp * np.asarray(w).reshape((1,) * ax + (n,) + (1,) * (2 - ax))
for _ in range(2):
    want = want * np.exp((0.5j * 0.05) * (1.0 - (want.real ** 2 + want.imag ** 2) / wp))
print(f"n={n}: product {t_plain:.4f} ms, +phase x1 {t_r1:.4f} (+{t_r1 - t_plain:.4f}), "
      f"+phase x2 {t_r2:.4f} (+{t_r2 - t_plain:.4f}), pointwise pass {t_pw:.4f} ms; "
      f"fused x2 parity {orc.rel_l2(got, want):.2e}")
