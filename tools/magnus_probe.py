"""Where does a device-expm Magnus step (k=256 c128) spend its time?"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2103_01691_b200 as km  # noqa: E402
from paper_2103_01691_b200 import _device as dv  # noqa: E402
from paper_2103_01691_b200.expm import matexp_device, prepare_device  # noqa: E402
from paper_2103_01691_b200.problems import hkmp_factors  # noqa: E402

DEV = torch.device("cuda", 0)
k, tau = 256, 1.0 / 32
b = km.hermite_basis(k)
u = dv.to_device(np.asfortranarray(np.random.default_rng(0).standard_normal((k,) * 3) + 0j), np.complex128, DEV)


def ev_time(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    t1 = time.perf_counter()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps, (t1 - t0) * 1e3 / reps


op = hkmp_factors(b, 0.3)
print("host factors build: %.3f ms" % (ev_time(lambda: hkmp_factors(b, 0.3))[1]))
A = tau * op.factors[2]
print("one device expm (device ms, host-issue ms): %.3f %.3f" % ev_time(lambda: matexp_device(A)))
cache = prepare_device(op, tau)
print("tucker step with device cache: %.3f %.3f" % ev_time(lambda: km.step(cache, u)))
print("prepare_device (3 expm): %.3f %.3f" % ev_time(lambda: prepare_device(op, tau)))
print("full magnus step: %.3f %.3f" % ev_time(
    lambda: km.magnus_midpoint_step(lambda t: hkmp_factors(b, t), u, 0.1, tau, device_expm=True)))
from paper_2103_01691_b200 import tensor as _tensor  # noqa: E402
from paper_2103_01691_b200.kron import _cache_mats, _Operand  # noqa: E402


def general_path():
    c = prepare_device(hkmp_factors(b, 0.1 + 0.5 * tau), tau)
    return _tensor.run_tucker(u, _cache_mats(c, _Operand(u)))


print("magnus step through run_tucker (no StepPlan): %.3f %.3f" % ev_time(general_path))
print("full magnus step again: %.3f %.3f" % ev_time(
    lambda: km.magnus_midpoint_step(lambda t: hkmp_factors(b, t), u, 0.1, tau, device_expm=True)))

# the bench_configs sequence: 4 chained steps at s * tau (wall clock per step)
c0 = u
for label in ("chained, device expm", "chained, device expm (2nd)", "chained, host expm"):
    dev_flag = "device" in label
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x = c0
    times = []
    for s in range(4):
        ts = time.perf_counter()
        x = km.magnus_midpoint_step(lambda t: hkmp_factors(b, t), x, s * tau, tau, device_expm=dev_flag)
        torch.cuda.synchronize()
        times.append((time.perf_counter() - ts) * 1e3)
    print(label, "per step ms:", ["%.2f" % v for v in times])
