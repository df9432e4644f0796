"""Where does the GPE Strang step's time go? (plain exact step vs Strang step, pointwise pass alone)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2103_01691_b200 as km  # noqa: E402
from paper_2103_01691_b200 import _device as dv, _native  # noqa: E402
from paper_2103_01691_b200.problems import _gpe_op, weighted_vortex_state  # noqa: E402

dev = torch.device("cuda", 0)


def timeit(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


for n in (256, 512):
    grids, lin_op, weights = km.gpe_setup(n)
    psi = weighted_vortex_state(grids, weights)
    cache = km.prepare(lin_op, 0.1)
    p = dv.to_device(psi, np.complex128, dev)
    t_step = timeit(lambda: km.step(cache, p))
    t_gpe = timeit(lambda: km.gpe_strang_step(cache, weights, p, 0.1))
    w_dev = [dv.cached_vector(w, np.float64, dev) for w in weights]
    op = _gpe_op(p.shape, w_dev, 0.05)
    out = torch.empty_like(p)
    lib = _native.lib()
    t_pw = timeit(lambda: lib.km_pointwise(p.data_ptr(), out.data_ptr(), _native.KM_C128, p.numel(),
                                           ctypes.byref(op), dv.stream_ptr(dev)))
    print(f"n={n}: step {t_step:.3f} ms, gpe_strang {t_gpe:.3f} ms, pointwise pass {t_pw:.3f} ms "
          f"({2 * 16 * n**3 / t_pw / 1e6:.0f} GB/s)")
