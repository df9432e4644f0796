"""One launch of every kernel family, for an `ncu --set full` evidence capture.

    python tools/profile_kernels.py            # all cases
    python tools/profile_kernels.py c64 gpe    # selected cases

Cases: steps (64^3 x 10 persistent launch), matvec (256^3 Kronecker-sum matvec, accumulate
epilogues), gpe64 (256^3 GPE step from complex64: widening phase pass),
c128 (256^3 exact step, TMA DMMA kernel), c64 (256^3 complex64 step:
prep_planes + tcgen05 kernel), small (64^3 complex128 step, cp.async DMMA
kernel), pipe (1024^2 float64 step), gpe (256^3 GPE Strang step: pointwise
pre pass + products with the fused phase epilogue), norm (256^3 two and
weighted_two norms).  Inputs are built and uploaded before the first kernel.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2103_01691_b200 as km  # noqa: E402
from paper_2103_01691_b200 import _device as dv  # noqa: E402

DEV = torch.device("cuda", 0)


def crand(shape, dtype=np.complex128, seed=0):
    rng = np.random.default_rng(seed)
    return np.asfortranarray((rng.standard_normal(shape) + 1j * rng.standard_normal(shape)).astype(dtype))


def schrod(n, dtype=np.complex128):
    d2 = km.heat_factors(n, 2).factors[0]
    c = km.prepare(km.KroneckerOp((1j * d2,) * 3), 0.01)
    return km.PropagatorCache(0.01, tuple(e.astype(dtype) for e in c.exps))


def case_c128():
    cache, t = schrod(256), dv.to_device(crand((256,) * 3), np.complex128, DEV)
    return lambda: km.step(cache, t)


def case_c64():
    cache, t = schrod(256, np.complex64), dv.to_device(crand((256,) * 3, np.complex64), np.complex64, DEV)
    return lambda: km.step(cache, t)


def case_small():
    cache, t = schrod(64), dv.to_device(crand((64,) * 3), np.complex128, DEV)
    return lambda: km.step(cache, t)


def case_pipe():
    op = km.pipeflow_factors(1024)
    cache = km.prepare(op, 4.0 / 16)
    rho, z = km.fd.pipeflow_grids(1024)
    c0 = np.asfortranarray(np.exp(-8.0 * (rho.points - 2.55) ** 2)[:, None] * np.exp(-8.0 * (z.points - 1.5) ** 2)[None, :])
    t = dv.to_device(c0, np.float64, DEV)
    return lambda: km.step(cache, t)


def case_gpe():
    _, lin_op, weights = km.gpe_setup(256)
    cache = km.prepare(lin_op, 0.1)
    t = dv.to_device(crand((256,) * 3), np.complex128, DEV)
    return lambda: km.gpe_strang_step(cache, weights, t, 0.1)


def case_slab8():
    """Rank 0's products of the 256^3 state split over 8 GPUs (two-half schedule, stream-K tail), one step."""
    from paper_2103_01691_b200 import dist

    u = crand((256,) * 3)
    d2 = km.heat_factors(256, 2).factors[0]
    cache = km.prepare(km.KroneckerOp((1j * d2,) * 3), 0.01)
    g = dist.VirtualSlabGroup(u, cache, DEV, 8)
    r0 = g.ranks[0]
    return lambda: (r0.begin_step(), r0.end_step())


def case_norm():
    t = dv.to_device(crand((256,) * 3), np.complex128, DEV)
    w = [np.linspace(0.5, 1.5, 256)] * 3
    return lambda: (km.norm(t, "two"), km.norm(t, "weighted_two", weights=w))


def case_steps():
    """64^3 complex128 x 10 steps in one persistent launch (km_steps_small, opt-in)."""
    from paper_2103_01691_b200 import dist

    cache, t = schrod(64), dv.to_device(crand((64,) * 3), np.complex128, DEV)
    st = dist.LocalStepper(t, cache.device_exps((np.complex128,) * 3, DEV))
    return lambda: st.run(10, persistent=True)


def case_paired():
    """64^3 complex128 x 2 steps as km_steps_paired's three fused launches (plane, pencil, plane)."""
    from paper_2103_01691_b200 import dist

    cache, t = schrod(64), dv.to_device(crand((64,) * 3), np.complex128, DEV)
    st = dist.LocalStepper(t, cache.device_exps((np.complex128,) * 3, DEV))
    return lambda: st.run(2)


def case_matvec():
    """256^3 complex128 Kronecker-sum matvec: 3 products, the last two accumulating in the epilogue."""
    d2 = km.heat_factors(256, 2).factors[0]
    op = km.KroneckerOp((1j * d2,) * 3)
    t = dv.to_device(crand((256,) * 3), np.complex128, DEV)
    return lambda: km.matvec(op, t)


def case_gpe64():
    """256^3 GPE Strang step from a complex64 state: the widening opening phase (float32 density)."""
    _, lin_op, weights = km.gpe_setup(256)
    cache = km.prepare(lin_op, 0.1)
    t = dv.to_device(crand((256,) * 3, np.complex64), np.complex64, DEV)
    return lambda: km.gpe_strang_step(cache, weights, t, 0.1)


CASES = {"c128": case_c128, "c64": case_c64, "small": case_small, "pipe": case_pipe, "gpe": case_gpe,
         "norm": case_norm, "slab8": case_slab8, "steps": case_steps, "matvec": case_matvec, "gpe64": case_gpe64,
         "paired": case_paired}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    runs = [CASES[n]() for n in names]  # all uploads first
    torch.cuda.synchronize()
    for run in runs:
        run()
    torch.cuda.synchronize()
    print("ok", names)
