"""Configuration 1 and neighbours: `steps` exact steps of an n^3 complex128 cube.

    python tools/steps_probe.py [steps]

Per n: the persistent dataflow launch (km_steps_small via LocalStepper.run), the
per-step km_tucker launches replayed as a CUDA graph (the round-1 path), and the
achieved fraction of the measured DMMA peak (37.14 TFLOP/s) at 8 flop per complex MAC.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2103_01691_b200 as km  # noqa: E402
from oracle import kronmode_oracle as orc  # noqa: E402
from paper_2103_01691_b200 import _device as dv  # noqa: E402
from paper_2103_01691_b200 import dist  # noqa: E402

DEV = torch.device("cuda", 0)
PEAK = 37.14e12
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 10


def dev_time(fn, reps=50, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


for n in (32, 64, 96):
    rng = np.random.default_rng(0)
    u = np.asfortranarray(rng.standard_normal((n,) * 3) + 1j * rng.standard_normal((n,) * 3))
    d2 = km.heat_factors(n, 2).factors[0]
    cache = km.prepare(km.KroneckerOp((1j * d2,) * 3), 0.01)
    mats = cache.device_exps((np.complex128,) * 3, DEV)
    flop = 8 * 3 * n**4 * steps
    st = dist.LocalStepper(dv.to_device(u, np.complex128, DEV), mats)
    ms_p = dev_time(lambda: st.run(steps, persistent=True))
    st2 = dist.LocalStepper(dv.to_device(u, np.complex128, DEV), mats)
    for _ in range(3):
        st2.step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(steps):
                st2.step()
    torch.cuda.synchronize()
    ms_g = dev_time(g.replay)
    st3 = dist.LocalStepper(dv.to_device(u, np.complex128, DEV), mats)
    st3.run(steps, persistent=True)
    want = u
    for _ in range(steps):
        want = orc.step(cache.exps, want)
    err = orc.rel_l2(dv.to_host(st3.state), want)
    print(f"n={n} x {steps} steps: persistent {ms_p * 1e3:.1f} us ({flop / (ms_p * 1e-3) / PEAK:.3f} of DMMA peak), "
          f"per-step graph {ms_g * 1e3:.1f} us ({flop / (ms_g * 1e-3) / PEAK:.3f}); parity {err:.2e}", flush=True)
