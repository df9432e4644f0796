"""Per-tile timeline of km_steps_small (a KMB_STEPS_TRACE build: build/tmp_trace/libkmb200.so).

    KMB200_LIB=build/tmp_trace/libkmb200.so python tools/steps_trace.py [n] [steps]

Stamps per tile (globaltimer, ns): start, dependencies satisfied, A staged, MMAs done,
published.  Prints per product: first start / last publish, and the mean phase times.
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2103_01691_b200 as km  # noqa: E402
from paper_2103_01691_b200 import _device as dv, _native, dist  # noqa: E402

DEV = torch.device("cuda", 0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
rng = np.random.default_rng(0)
u = np.asfortranarray(rng.standard_normal((n,) * 3) + 1j * rng.standard_normal((n,) * 3))
d2 = km.heat_factors(n, 2).factors[0]
cache = km.prepare(km.KroneckerOp((1j * d2,) * 3), 0.01)
mats = cache.device_exps((np.complex128,) * 3, DEV)
st = dist.LocalStepper(dv.to_device(u, np.complex128, DEV), mats)
tiles = (n // 32) * n * (n // 32)
trace = torch.zeros(3 * steps * tiles * 6, dtype=torch.int64, device=DEV)
lib = _native.lib()
lib.km_steps_small_trace.argtypes = [ctypes.c_void_p]
st.run(steps)  # warm
lib.km_steps_small_trace(trace.data_ptr())
torch.cuda.synchronize()
st.run(steps)
torch.cuda.synchronize()
lib.km_steps_small_trace(None)
tr = trace.cpu().numpy().reshape(-1, 6)
t0 = tr[:, 0].min()
for p in range(3 * steps):
    x = tr[p * tiles:(p + 1) * tiles]
    print(f"product {p}: first start {(x[:, 0].min() - t0) / 1e3:7.2f} us, last start {(x[:, 0].max() - t0) / 1e3:7.2f}, "
          f"last publish {(x[:, 4].max() - t0) / 1e3:7.2f}; mean wait {np.mean(x[:, 1] - x[:, 0]) / 1e3:.2f}, "
          f"A {np.mean(x[:, 2] - x[:, 1]) / 1e3:.2f}, mma {np.mean(x[:, 3] - x[:, 2]) / 1e3:.2f}, "
          f"store+publish {np.mean(x[:, 4] - x[:, 3]) / 1e3:.2f} us; CTAs {len(set((x[:, 5] >> 32).tolist()))}")
