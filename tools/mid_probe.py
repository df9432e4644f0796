"""Mid-size exact steps (96^3 .. 192^3, rectangular, 2048^2): device time per step (LocalStepper,
CUDA events) and per-direction launch times, for the cp.async / TMA / stream-K kernel choice.

    python tools/mid_probe.py
"""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2103_01691_b200 as km
from paper_2103_01691_b200 import _device as dv, dist
dev = torch.device("cuda", 0)
for shape in [(96,)*3, (128,)*3, (160,)*3, (192,)*3, (128, 128, 512), (512, 512, 16), (2048, 2048)]:
    rng = np.random.default_rng(0)
    u = np.asfortranarray(rng.standard_normal(shape) + 1j * rng.standard_normal(shape))
    mats = [((rng.standard_normal((n, n)) + 1j*rng.standard_normal((n, n)))/np.sqrt(n)) for n in shape]
    cache = km.PropagatorCache(0.1, tuple(mats))
    st = dist.LocalStepper(dv.to_device(u, np.complex128, dev), cache.device_exps((np.complex128,)*len(shape), dev))
    for _ in range(3): st.step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): st.step()
    e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1) / 10
    N = np.prod(shape); flop = 8 * N * sum(shape)
    print(f"{shape}: {ms*1e3:.1f} us/step, {flop/ms/1e9:.1f} TFLOP/s, launches {[round(x*1e3,1) for x in st.time_launches(10)]}")
