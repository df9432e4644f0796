"""Configuration 4 (TD-potential Strang, 256^3 c128 on the Gauss-Hermite grid): device time of
tdpot_strang_step (CUDA events, device-resident state) and parity against the oracle restatement.

    python tools/tdpot_probe.py [k]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2103_01691_b200 as km  # noqa: E402
from oracle import kronmode_oracle as orc  # noqa: E402
from paper_2103_01691_b200 import _device as dv  # noqa: E402
from paper_2103_01691_b200.hermite import physical_propagator  # noqa: E402
from paper_2103_01691_b200.problems import schrodinger_initial_state  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 256
b = km.hermite_basis(k)
tau = 0.02
p = physical_propagator(b, tau)
cache = km.PropagatorCache(tau, (p, p, p))
psi = schrodinger_initial_state((b.nodes,) * 3)
dev = torch.device("cuda", 0)
t = dv.to_device(psi, np.complex128, dev)
for _ in range(3):
    km.tdpot_strang_step(cache, b.nodes, t, 0.3, tau)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for s in range(10):
    km.tdpot_strang_step(cache, b.nodes, t, 0.3 + s * tau, tau)
e1.record()
e1.synchronize()
ms = e0.elapsed_time(e1) / 10
got = dv.to_host(km.tdpot_strang_step(cache, b.nodes, t, 0.3, tau))
want = orc.tdpot_strang_step(cache.exps, b.nodes, psi, 0.3, tau)
print(f"k={k}: tdpot_strang_step {ms:.3f} ms, {8 * 3 * k**4 / ms / 1e9:.1f} TFLOP/s, rel_l2 {orc.rel_l2(got, want):.2e}")
