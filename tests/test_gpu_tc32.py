"""GPU: complex64 products on the tcgen05 (kind::tf32, 3xTF32 split) kernel against
the oracle (the reference's own complex64 arithmetic) and the complex128 oracle."""

import numpy as np
import pytest

import paper_2103_01691_b200 as km
from oracle import kronmode_oracle as orc
from paper_2103_01691_b200 import _native

pytestmark = pytest.mark.gpu


def crand(rng, shape, dt=np.complex64):
    return np.asfortranarray((rng.standard_normal(shape) + 1j * rng.standard_normal(shape)).astype(dt))


CASES = [((128, 128, 128), 1, 128), ((128, 128, 128), 2, 128), ((128, 128, 128), 3, 128),
         ((200, 96, 64), 1, 200), ((200, 96, 64), 3, 64), ((128, 128, 128), 3, 100),
         ((256, 256, 256), 1, 256), ((256, 256, 256), 2, 256), ((256, 256, 256), 3, 256)]


@pytest.mark.parametrize("shape,mu,m", CASES)
def test_c64_products_vs_oracle(shape, mu, m):
    rng = np.random.default_rng(sum(shape) + mu + m)
    u = crand(rng, shape)
    mat = ((rng.standard_normal((m, shape[mu - 1])) + 1j * rng.standard_normal((m, shape[mu - 1])))
           / np.sqrt(shape[mu - 1])).astype(np.complex64)
    got = km.mu_mode_product(u, mat, mu)
    assert got.dtype == np.complex64
    want64 = orc.mu_mode_product(u, mat, mu)
    want128 = orc.mu_mode_product(u.astype(np.complex128), mat.astype(np.complex128), mu)
    e64, e128 = orc.rel_l2(got, want64), orc.rel_l2(got, want128)
    assert e64 <= 1e-5, e64
    assert e128 <= 1e-5, e128


def test_c64_step_256_vs_oracle_and_dmma():
    n = 256
    rng = np.random.default_rng(0)
    u = crand(rng, (n,) * 3)
    d2 = km.heat_factors(n, 2).factors[0]
    c128 = km.prepare(km.KroneckerOp((1j * d2,) * 3), 0.01)
    cache = km.PropagatorCache(0.01, tuple(e.astype(np.complex64) for e in c128.exps))
    got = km.step(cache, u)
    want = orc.step(cache.exps, u)
    assert orc.rel_l2(got, want) <= 1e-5
    lib = _native.lib()
    try:
        _native.check(lib.km_set_kernel_policy(_native.POLICY_NO_TMA))
        dmma = km.step(cache, u)
    finally:
        _native.check(lib.km_set_kernel_policy(_native.POLICY_AUTO))
    assert orc.rel_l2(got, dmma) <= 1e-5


LONG = [((384, 64, 8), 1), ((512, 128, 8), 1), ((1024, 64, 4), 1), ((128, 1024, 8), 2), ((128, 8, 1024), 3),
        ((256, 8, 640), 3), ((128, 8, 520), 3)]


@pytest.mark.parametrize("shape,mu", LONG)
@pytest.mark.parametrize("halves", [True, False])
def test_long_contractions(shape, mu, halves):
    """K' > 512.  Up to K' = 1024 the default is two accumulation chains of <= 512 k' per tile
    summed in fp32 (HALVES): the error stays at the K' = 512 level of the production kernel
    (measured 3.7e-6).  Beyond that, and for K' <= 1024 under KM_POLICY_NO_TC_HALVES, the
    chunked kernel (fresh TMEM accumulator every 64 k', fp32 drain) keeps it lower."""
    rng = np.random.default_rng(sum(shape) + mu)
    u = crand(rng, shape)
    n = shape[mu - 1]
    kp = 2 * n if mu == 1 else n
    mat = ((rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / np.sqrt(n)).astype(np.complex64)
    lib = _native.lib()
    try:
        if not halves:
            _native.check(lib.km_set_kernel_policy(_native.POLICY_NO_TC_HALVES))
        got = km.mu_mode_product(u, mat, mu)
    finally:
        _native.check(lib.km_set_kernel_policy(_native.POLICY_AUTO))
    want128 = orc.mu_mode_product(u.astype(np.complex128), mat.astype(np.complex128), mu)
    want64 = orc.mu_mode_product(u, mat, mu)
    e128, e64 = orc.rel_l2(got, want128), orc.rel_l2(got, want64)
    assert e128 <= (5e-6 if halves and kp <= 1024 else 2e-6), e128
    assert e64 <= 1e-5, e64


@pytest.mark.parametrize("mu", [1, 2, 3])
def test_complex64_state_with_real_float32_factor_on_tcgen05(mu):
    """complex64 x float32 (the single-precision Hermite transforms): numpy promotes the real
    factor to complex64 (tensor.py:121-123), so the product runs on the tcgen05 kernel with the
    promoted factor; parity against the reference's own complex64 arithmetic."""
    import torch

    from conftest import kernels_launched
    from paper_2103_01691_b200 import _device as dv

    n = 128
    rng = np.random.default_rng(mu)
    u = np.asfortranarray((rng.standard_normal((n,) * 3) + 1j * rng.standard_normal((n,) * 3)).astype(np.complex64))
    phi = (rng.standard_normal((n, n)) / np.sqrt(n)).astype(np.float32)
    t = dv.to_device(u, np.complex64, torch.device("cuda", 0))
    got, names = kernels_launched(lambda: km.mu_mode_product(t, phi, mu))
    assert names is None or any("mumode_tc32" in x for x in names), names
    got = dv.to_host(got)
    assert got.dtype == np.complex64
    want = orc.mu_mode_product(u, phi, mu)
    assert orc.rel_l2(got, want) <= 1e-5


@pytest.mark.parametrize("shape", [(256, 256, 128), (160, 256, 256), (2, 4200, 1000), (4096, 2048)])
def test_float32_products_pair_fibers_on_tcgen05(shape):
    """float32 x float32: directions with an even n_left read two real fibers as one complex64
    fiber on the tcgen05 kernel (direction 1 stays on DMMA); parity with the reference's float32
    arithmetic within the single-precision bar, and the tcgen05 kernel actually ran."""
    from conftest import kernels_launched
    from paper_2103_01691_b200 import _device as dv

    rng = np.random.default_rng(sum(shape))
    u = np.asfortranarray(rng.standard_normal(shape).astype(np.float32))
    mats = [(rng.standard_normal((n, n)) / np.sqrt(n)).astype(np.float32) for n in shape]
    t = dv.to_device(u, np.float32, dv.device())
    got, names = kernels_launched(lambda: km.tucker(t, mats))
    assert dv.np_dtype(got.dtype) == np.float32
    want = orc.tucker(u.astype(np.float64), [m.astype(np.float64) for m in mats])
    assert orc.rel_l2(dv.to_host(got), want) <= 1e-5
    if names is not None:
        assert any("mumode_tc32" in n for n in names)
    host = km.tucker(u, mats)  # numpy in, numpy out (the host pipeline or the same loop)
    assert host.dtype == np.float32 and orc.rel_l2(host, want) <= 1e-5
