"""GPU: km_steps_small — many exact steps of a small complex128 cube in one persistent
launch (the sweeps of all steps as a dataflow of tiles, kmb200_small.cuh) — against the
oracle's step loop (kron.py:110-121 applied `steps` times) and the per-step launches."""

import ctypes

import numpy as np
import pytest

import paper_2103_01691_b200 as km
from oracle import kronmode_oracle as orc
from paper_2103_01691_b200 import _device as dv
from paper_2103_01691_b200 import _native, dist

pytestmark = pytest.mark.gpu


def crand(rng, shape):
    return np.asfortranarray(rng.standard_normal(shape) + 1j * rng.standard_normal(shape))


@pytest.mark.parametrize("shape,steps", [((64, 64, 64), 10), ((64, 64, 64), 1), ((32, 32, 32), 7),
                                         ((96, 96, 96), 3), ((32, 64, 96), 4), ((96, 32, 64), 2)])
def test_persistent_steps_match_oracle_and_step_loop(shape, steps):
    import torch

    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(sum(shape) + steps)
    u = crand(rng, shape)
    exps = []
    for n in shape:
        d2 = km.heat_factors(n, 2).factors[0]
        exps.append(km.prepare(km.KroneckerOp((1j * d2,)), 0.01).exps[0])
    cache = km.PropagatorCache(0.01, tuple(exps))
    mats = cache.device_exps((np.complex128,) * 3, dev)
    st = dist.LocalStepper(dv.to_device(u, np.complex128, dev), mats)
    assert st._steps_workspace(steps) is not None
    st.run(steps, persistent=True)
    got = dv.to_host(st.state)
    want = u
    for _ in range(steps):
        want = orc.step(cache.exps, want)
    assert orc.rel_l2(got, want) <= 1e-12
    ref = dist.LocalStepper(dv.to_device(u, np.complex128, dev), mats)
    for _ in range(steps):
        ref.step()
    assert orc.rel_l2(got, dv.to_host(ref.state)) <= 1e-13
    # the kernel ran (and only it): one launch for all the sweeps
    from conftest import kernels_launched

    st2 = dist.LocalStepper(dv.to_device(u, np.complex128, dev), mats)
    _, names = kernels_launched(lambda: st2.run(steps, persistent=True))
    if names is not None:
        assert sum("mumode_steps_kernel" in x for x in names) == 1, names
        assert not any("mumode_kernel" in x or "mumode_tma_kernel" in x for x in names)


def test_repeated_runs_reuse_counters():
    """The dependency counters are re-zeroed per launch: back-to-back runs on one stream."""
    import torch

    dev = torch.device("cuda", 0)
    n = 64
    rng = np.random.default_rng(3)
    u = crand(rng, (n,) * 3)
    d2 = km.heat_factors(n, 2).factors[0]
    cache = km.prepare(km.KroneckerOp((1j * d2,) * 3), 0.01)
    mats = cache.device_exps((np.complex128,) * 3, dev)
    st = dist.LocalStepper(dv.to_device(u, np.complex128, dev), mats)
    for _ in range(5):
        st.run(4, persistent=True)
    want = u
    for _ in range(20):
        want = orc.step(cache.exps, want)
    assert orc.rel_l2(dv.to_host(st.state), want) <= 1e-12


@pytest.mark.parametrize("shape", [(48, 64, 64), (128, 64, 64), (64, 64, 16)])
def test_ineligible_shapes_fall_back(shape):
    import torch

    lib = _native.lib()
    nb = ctypes.c_size_t()
    assert lib.km_steps_small_workspace_bytes(*shape, 3, ctypes.byref(nb)) == _native.KM_EINVAL
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(1)
    u = crand(rng, shape)
    mats_h = [np.asarray(km.prepare(km.KroneckerOp((1j * km.heat_factors(n, 2).factors[0],)), 0.01).exps[0])
              for n in shape]
    mats = [torch.from_numpy(np.ascontiguousarray(m)).to(dev) for m in mats_h]
    st = dist.LocalStepper(dv.to_device(u, np.complex128, dev), mats)
    assert st._steps_workspace(2) is None
    st.run(2, persistent=True)
    assert orc.rel_l2(dv.to_host(st.state), orc.step(mats_h, orc.step(mats_h, u))) <= 1e-12
