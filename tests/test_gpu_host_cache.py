"""GPU: the device copies of host factors (_device.cached_vector) follow the
host arrays: an in-place change, a recycled buffer or a different dtype view
is uploaded again, so mu_mode_product always sees the current values (the
reference multiplies by the array as it is at call time, tensor.py:129/139)."""

import numpy as np
import pytest

import paper_2103_01691_b200 as km
from oracle import kronmode_oracle as orc
from paper_2103_01691_b200 import _device as dv

pytestmark = pytest.mark.gpu


def test_in_place_change_of_a_factor_is_seen():
    rng = np.random.default_rng(3)
    u = np.asfortranarray(rng.standard_normal((16, 12, 8)) + 1j * rng.standard_normal((16, 12, 8)))
    mat = rng.standard_normal((12, 12)) + 1j * rng.standard_normal((12, 12))
    for mu_val in range(3):
        got = km.mu_mode_product(u, mat, 2)
        assert orc.rel_l2(got, orc.mu_mode_product(u, mat, 2)) <= 1e-14
        mat[mu_val, 5] += 1.0  # same buffer, new content
        mat[7, :] *= -0.5


def test_fortran_and_c_order_factors_and_weights():
    rng = np.random.default_rng(4)
    u = np.asfortranarray(rng.standard_normal((8, 8, 8)))
    mat = rng.standard_normal((8, 8))
    for m in (mat, np.asfortranarray(mat), mat.T, mat[:, ::-1]):
        got = km.mu_mode_product(u, m, 3)
        assert orc.rel_l2(got, orc.mu_mode_product(u, m, 3)) <= 1e-14


def test_cache_hit_returns_the_same_device_copy():
    import torch

    dev = torch.device("cuda", 0)
    a = np.arange(64.0).reshape(8, 8)
    t1 = dv.cached_vector(a, np.float64, dev)
    t2 = dv.cached_vector(a, np.float64, dev)
    assert t1 is t2
    a[0, 0] = -1.0
    t3 = dv.cached_vector(a, np.float64, dev)
    assert t3 is not t1 and float(t3[0, 0]) == -1.0
    # same buffer, another target dtype: a separate entry
    t4 = dv.cached_vector(a, np.float32, dev)
    assert t4.dtype == torch.float32 and float(t4[0, 0]) == -1.0


def test_step_plan_reuse_across_streams_and_dtypes():
    """kron.step's prebuilt call (StepPlan): correct on repeated calls, on a second stream (its own
    scratch buffer), for a float32 state with complex128 factors (no plan: the general path
    promotes), and the flop tally still counts every product."""
    import numpy as np
    import torch

    import paper_2103_01691_b200 as km
    from oracle import kronmode_oracle as orc
    from paper_2103_01691_b200 import _device as dv

    dev = torch.device("cuda", 0)
    n = 24
    rng = np.random.default_rng(12)
    u = np.asfortranarray(rng.standard_normal((n,) * 3) + 1j * rng.standard_normal((n,) * 3))
    d2 = km.heat_factors(n, 2).factors[0]
    cache = km.prepare(km.KroneckerOp((1j * d2,) * 3), 0.01)
    t = dv.to_device(u, np.complex128, dev)
    with km.count_flops() as fc:
        a = km.step(cache, t)
        b = km.step(cache, a)
    assert fc.macs == 2 * 3 * n**4
    want1 = orc.step(cache.exps, u)
    want2 = orc.step(cache.exps, want1)
    assert orc.rel_l2(dv.to_host(a), want1) <= 1e-12 and orc.rel_l2(dv.to_host(b), want2) <= 1e-12
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        c = km.step(cache, t)
        d = km.step(cache, c)
    s.synchronize()
    assert np.array_equal(dv.to_host(c), dv.to_host(a)) and np.array_equal(dv.to_host(d), dv.to_host(b))
    t32 = dv.to_device(u.real.astype(np.float32), np.float32, dev)
    r = km.step(cache, t32)
    assert dv.np_dtype(r.dtype) == np.complex128
    assert orc.rel_l2(dv.to_host(r), orc.step(cache.exps, u.real.astype(np.float32))) <= 1e-12


def test_step_plan_does_not_pin_large_scratch():
    """A state whose Tucker scratch exceeds StepPlan.KEEP_WS_BYTES takes it from torch's allocator
    per call: the cache keeps no state-sized buffer alive, and the result is unchanged."""
    import numpy as np
    import torch

    import paper_2103_01691_b200 as km
    from oracle import kronmode_oracle as orc
    from paper_2103_01691_b200 import _device as dv
    from paper_2103_01691_b200.tensor import StepPlan

    dev = torch.device("cuda", 0)
    n = 160  # 160^3 complex128: 65.5 MB of scratch
    rng = np.random.default_rng(13)
    u = np.asfortranarray(rng.standard_normal((n,) * 3) + 1j * rng.standard_normal((n,) * 3))
    d2 = km.heat_factors(n, 2).factors[0]
    cache = km.prepare(km.KroneckerOp((1j * d2,) * 3), 0.01)
    t = dv.to_device(u, np.complex128, dev)
    a = km.step(cache, t)
    b = km.step(cache, t)
    (plan,) = cache._plans.values()
    assert plan.ok and plan.plan[7] > StepPlan.KEEP_WS_BYTES and not plan.ws
    assert torch.equal(a, b)
    assert orc.rel_l2(dv.to_host(a), orc.step(cache.exps, u)) <= 1e-12


def test_long_step_loops_hold_memory_flat():
    """Hundreds of public-API steps (64^3 fused planes, 128^3 products, a new Magnus cache per
    step) leave torch's allocated device memory where the first steps put it: no per-call growth
    from the prebuilt-call memo, the stream workspaces or the factor caches."""
    import numpy as np
    import torch

    import paper_2103_01691_b200 as km
    from paper_2103_01691_b200 import _device as dv
    from paper_2103_01691_b200.problems import hkmp_factors

    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(14)
    for n in (64, 128):
        d2 = km.heat_factors(n, 2).factors[0]
        cache = km.prepare(km.KroneckerOp((1j * d2,) * 3), 0.01)
        u = dv.to_device(np.asfortranarray(rng.standard_normal((n,) * 3) + 0j), np.complex128, dev)
        for _ in range(5):
            u = km.step(cache, u)
        torch.cuda.synchronize()
        base = torch.cuda.memory_allocated(dev)
        for _ in range(300):
            u = km.step(cache, u)
        torch.cuda.synchronize()
        assert torch.cuda.memory_allocated(dev) <= base
    b = km.hermite_basis(32)
    c = dv.to_device(np.asfortranarray(rng.standard_normal((32,) * 3) + 0j), np.complex128, dev)
    for s in range(3):
        c = km.magnus_midpoint_step(lambda t: hkmp_factors(b, t), c, 0.01 * s, 0.01, device_expm=True)
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated(dev)
    for s in range(100):
        c = km.magnus_midpoint_step(lambda t: hkmp_factors(b, t), c, 0.01 * s, 0.01, device_expm=True)
    torch.cuda.synchronize()
    assert torch.cuda.memory_allocated(dev) <= base
