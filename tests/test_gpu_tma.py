"""GPU: the warp-specialised TMA complex128 kernel (kmb200_tma.cuh) against the
oracle and against the cp.async kernel (km_set_kernel_policy), including
ragged M/N/K tails, the fused phase epilogue and the blocked (slab) layouts."""

import numpy as np
import pytest

import paper_2103_01691_b200 as km
from oracle import kronmode_oracle as orc
from paper_2103_01691_b200 import _native

pytestmark = pytest.mark.gpu


def crand(rng, shape):
    return np.asfortranarray(rng.standard_normal(shape) + 1j * rng.standard_normal(shape))


def both_policies(fn):
    lib = _native.lib()
    try:
        a = fn()
        _native.check(lib.km_set_kernel_policy(_native.POLICY_NO_TMA))
        b = fn()
    finally:
        _native.check(lib.km_set_kernel_policy(_native.POLICY_AUTO))
    return a, b


@pytest.mark.parametrize("shape,mu", [((264, 300, 40), 1), ((128, 200, 104), 2), ((128, 200, 104), 3),
                                      ((256, 256, 256), 1), ((256, 256, 256), 2), ((256, 256, 256), 3)])
def test_tma_products_with_tails(shape, mu):
    rng = np.random.default_rng(sum(shape) + mu)
    u = crand(rng, shape)
    n = shape[mu - 1]
    mat = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    import torch

    from paper_2103_01691_b200 import _device as dv

    t = dv.to_device(u, np.complex128, torch.device("cuda", 0))
    a, b = both_policies(lambda: dv.to_host(km.mu_mode_product(t, mat, mu)))
    want = orc.mu_mode_product(u, mat, mu)
    assert orc.rel_l2(a, want) <= 1e-13
    assert orc.rel_l2(b, want) <= 1e-13


def test_tma_gpe_epilogue():
    n = 256
    grids, lin_op, weights = km.gpe_setup(n)
    from paper_2103_01691_b200.problems import weighted_vortex_state

    psi = weighted_vortex_state(grids, weights)
    cache = km.prepare(lin_op, 0.1)
    a, b = both_policies(lambda: km.gpe_strang_step(cache, weights, psi, 0.1))
    want = orc.gpe_strang_step(cache.exps, weights, psi, 0.1)
    assert orc.rel_l2(a, want) <= 1e-12 and orc.rel_l2(b, want) <= 1e-12


@pytest.mark.parametrize("steps", [1, 2])
def test_tma_blocked_layouts_virtual_ranks(steps):
    import torch

    from paper_2103_01691_b200 import _device as dv
    from paper_2103_01691_b200 import dist

    dev = torch.device("cuda", 0)
    n = 256
    u = crand(np.random.default_rng(7), (n,) * 3)
    d2 = km.heat_factors(n, 2).factors[0]
    cache = km.prepare(km.KroneckerOp((1j * d2,) * 3), 0.01)
    grp = dist.VirtualSlabGroup(u, cache, dev, 2)  # 256/2 = 128-row blocks: TMA-eligible
    for _ in range(steps):
        grp.step()
    ref = dist.LocalStepper(dv.to_device(u, np.complex128, dev), cache.device_exps((np.complex128,) * 3, dev))
    for _ in range(steps):
        ref.step()
    assert orc.rel_l2(grp.gather(), dv.to_host(ref.state)) <= 1e-12


@pytest.mark.parametrize("shape,mu", [((264, 300, 40), 1), ((128, 200, 104), 2), ((128, 200, 104), 3),
                                      ((256, 256, 256), 1), ((256, 256, 256), 2), ((256, 256, 256), 3)])
def test_tma_real_factor_products(shape, mu):
    """complex tensor x real factor (the Hermite transforms' shape of product)"""
    import torch

    from paper_2103_01691_b200 import _device as dv

    rng = np.random.default_rng(sum(shape) * 3 + mu)
    u = crand(rng, shape)
    n = shape[mu - 1]
    mat = rng.standard_normal((n + 8, n))  # rectangular: m != n_mu
    t = dv.to_device(u, np.complex128, torch.device("cuda", 0))
    a, b = both_policies(lambda: dv.to_host(km.mu_mode_product(t, mat, mu)))
    want = orc.mu_mode_product(u, mat, mu)
    assert orc.rel_l2(a, want) <= 1e-13
    assert orc.rel_l2(b, want) <= 1e-13


@pytest.mark.parametrize("shape,mu,cl", [((1024, 1024), 1, False), ((1024, 1024), 2, False),
                                         ((264, 300, 40), 1, True), ((256, 256, 256), 2, True),
                                         ((256, 256, 256), 3, False), ((128, 200, 104), 3, False)])
def test_tma_real_tensor_products(shape, mu, cl):
    """real tensor x real factor (pipe flow) and real tensor x complex factor"""
    import torch

    from paper_2103_01691_b200 import _device as dv

    rng = np.random.default_rng(sum(shape) * 5 + mu)
    u = np.asfortranarray(rng.standard_normal(shape))
    n = shape[mu - 1]
    mat = rng.standard_normal((n, n))
    if cl:
        mat = mat + 1j * rng.standard_normal((n, n))
    t = dv.to_device(u, np.float64, torch.device("cuda", 0))
    a, b = both_policies(lambda: dv.to_host(km.mu_mode_product(t, mat, mu)))
    want = orc.mu_mode_product(u, mat, mu)
    assert a.dtype == want.dtype
    assert orc.rel_l2(a, want) <= 1e-13
    assert orc.rel_l2(b, want) <= 1e-13
