"""GPU: the stream-K tail of the TMA kernel (kmb200_tma.cuh, StreamK) against
whole-tile scheduling (KM_POLICY_NO_STREAMK) and the oracle.

Tile counts cover: fewer tiles than SMs (all stream-K), a partial last wave
(whole waves + stream-K over the last two), exact multiples of the SM count
(no stream-K), real and complex operands, the fused GPE epilogue, the
blocked slab layouts, and repeated launches (per-launch epochs).
"""

import numpy as np
import pytest

import paper_2103_01691_b200 as km
from oracle import kronmode_oracle as orc
from paper_2103_01691_b200 import _device as dv
from paper_2103_01691_b200 import _native

pytestmark = pytest.mark.gpu


def crand(rng, shape):
    return np.asfortranarray(rng.standard_normal(shape) + 1j * rng.standard_normal(shape))


def policies(fn):
    """fn() with stream-K (AUTO), then with whole tiles only."""
    lib = _native.lib()
    try:
        a = fn()
        _native.check(lib.km_set_kernel_policy(_native.POLICY_NO_STREAMK))
        b = fn()
    finally:
        _native.check(lib.km_set_kernel_policy(_native.POLICY_AUTO))
    return a, b


def dev(x):
    import torch

    return dv.to_device(x, x.dtype, torch.device("cuda", 0))


# (shape, mu) with 128x64 tiles on 148 SMs: (1024, 1024) has 128 tiles (< 148: all stream-K);
# 256^3 has 2048 = 13*148 + 124; the 256^2 x 32 slab has 256 = 148 + 108; (128, 64, 296)
# along direction 2 has 296 = 2*148 (whole waves, no stream-K)
CASES = [((1024, 1024), 1, False), ((1024, 1024), 2, False), ((1024, 1024), 1, True),
         ((256, 256, 256), 1, True), ((256, 256, 256), 3, True), ((256, 256, 32), 3, True),
         ((256, 256, 32), 1, True), ((256, 256, 64), 2, True), ((128, 64, 296), 2, True)]


@pytest.mark.parametrize("shape,mu,cplx", CASES)
def test_streamk_products(shape, mu, cplx):
    rng = np.random.default_rng(sum(shape) + mu)
    u = crand(rng, shape) if cplx else np.asfortranarray(rng.standard_normal(shape))
    n = shape[mu - 1]
    mat = rng.standard_normal((n, n)) + (1j * rng.standard_normal((n, n)) if cplx else 0)
    t = dev(u)
    a, b = policies(lambda: dv.to_host(km.mu_mode_product(t, mat, mu)))
    want = orc.mu_mode_product(u, mat, mu)
    assert orc.rel_l2(a, want) <= 1e-13
    assert orc.rel_l2(b, want) <= 1e-13
    assert orc.rel_l2(a, b) <= 1e-14


# real x complex mixes (Hermite transforms, complex pipe-flow variant) and a
# tile count where a tile spans three CTAs: (1024, 896) along direction 2 has
# 8 x 14 = 112 tiles (S/2 <= 112 < S), 112 * 64 / 148 = 48 k-blocks per CTA
MIX_CASES = [((1024, 1024), 1, "rc"), ((1024, 1024), 2, "rc"), ((1024, 1024), 2, "cr"),
             ((1024, 896), 2, "rr"), ((1024, 896), 2, "cc"), ((896, 1024), 1, "rc")]


@pytest.mark.parametrize("shape,mu,mix", MIX_CASES)
def test_streamk_mixed_dtypes(shape, mu, mix):
    rng = np.random.default_rng(sum(shape) + mu + len(mix))
    u = crand(rng, shape) if mix[0] == "c" else np.asfortranarray(rng.standard_normal(shape))
    n = shape[mu - 1]
    mat = rng.standard_normal((n, n)) + (1j * rng.standard_normal((n, n)) if mix[1] == "c" else 0)
    t = dev(u)
    a, b = policies(lambda: dv.to_host(km.mu_mode_product(t, mat, mu)))
    want = orc.mu_mode_product(u, mat, mu)
    assert orc.rel_l2(a, want) <= 1e-13
    assert orc.rel_l2(b, want) <= 1e-13
    assert orc.rel_l2(a, b) <= 1e-14


# beyond 4 waves stream-K runs only when the last wave wastes > 5 % of the slots:
# (160,160,160) has 200 x 3 = 600 tiles (4.05 waves, 19 % waste; K = 160) -> stream-K,
# (192,192,192) has 288 x 3 = 864 (5.84 waves, 2.7 %) -> whole tiles
@pytest.mark.parametrize("shape,mu", [((160, 160, 160), 1), ((160, 160, 160), 3), ((192, 192, 192), 3)])
def test_streamk_many_waves(shape, mu):
    rng = np.random.default_rng(sum(shape) + mu)
    u = crand(rng, shape)
    n = shape[mu - 1]
    mat = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    t = dev(u)
    a, b = policies(lambda: dv.to_host(km.mu_mode_product(t, mat, mu)))
    want = orc.mu_mode_product(u, mat, mu)
    assert orc.rel_l2(a, want) <= 1e-13
    assert orc.rel_l2(b, want) <= 1e-13
    assert orc.rel_l2(a, b) <= 1e-14


def test_streamk_repeated_launches_are_deterministic():
    rng = np.random.default_rng(7)
    u = dev(crand(rng, (256, 256, 32)))
    mat = rng.standard_normal((256, 256)) + 1j * rng.standard_normal((256, 256))
    outs = [dv.to_host(km.mu_mode_product(u, mat, 1)).copy() for _ in range(5)]
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])


def test_streamk_step_and_gpe_epilogue():
    n = 256
    grids, lin_op, weights = km.gpe_setup(n)
    from paper_2103_01691_b200.problems import weighted_vortex_state

    psi = dev(weighted_vortex_state(grids, weights))
    cache = km.prepare(lin_op, 0.1)
    a, b = policies(lambda: dv.to_host(km.gpe_strang_step(cache, weights, psi, 0.1)))
    want = orc.gpe_strang_step(cache.exps, weights, dv.to_host(psi), 0.1)
    assert orc.rel_l2(a, want) <= 1e-12 and orc.rel_l2(b, want) <= 1e-12


@pytest.mark.parametrize("P", [4, 8])
def test_streamk_slab_layouts(P):
    """The virtual-rank slab decomposition (blocked split layouts) with stream-K tails."""
    import torch

    from paper_2103_01691_b200 import dist

    n = 256
    rng = np.random.default_rng(P)
    u = crand(rng, (n,) * 3)
    d2 = km.heat_factors(n, 2).factors[0]
    cache = km.prepare(km.KroneckerOp((1j * d2,) * 3), 0.01)

    def run():
        g = dist.VirtualSlabGroup(u, cache, torch.device("cuda", 0), P)
        for _ in range(2):
            g.step()
        return g.gather()

    a, b = policies(run)
    want = orc.step(cache.exps, orc.step(cache.exps, u))
    assert orc.rel_l2(a, want) <= 1e-12 and orc.rel_l2(b, want) <= 1e-12


@pytest.mark.parametrize("seed", range(6))
def test_random_large_shapes_vs_oracle(seed):
    """Ragged shapes large enough for the persistent TMA kernel (and, where the tile count
    lands between one and four waves, its stream-K tail): every direction, against the oracle."""
    rng = np.random.default_rng(100 + seed)
    n1 = int(rng.choice([128, 256]))  # fiber-contiguous layouts need n_left % 128 == 0
    shape = (n1, int(rng.integers(40, 300)) // 8 * 8, int(rng.integers(40, 200)) // 8 * 8)
    u = crand(rng, shape)
    t = dev(u)
    for mu in (1, 2, 3):
        n = shape[mu - 1]
        m = int(rng.integers(n // 2, n + 40))
        mat = rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n))
        a, b = policies(lambda: dv.to_host(km.mu_mode_product(t, mat, mu)))
        want = orc.mu_mode_product(u, mat, mu)
        assert orc.rel_l2(a, want) <= 1e-13, (shape, mu, m)
        assert orc.rel_l2(b, want) <= 1e-13, (shape, mu, m)


@pytest.mark.parametrize("seed", range(6))
def test_random_large_real_shapes_vs_oracle(seed):
    """As above for real tensors with real or complex factors (the 64-B-swizzled real tiles, the
    real x real producer warp): k extents with a half k-block tail (K % 16 == 8), ragged factor
    row counts, every direction, stream-K and whole tiles."""
    rng = np.random.default_rng(200 + seed)
    n1 = int(rng.choice([128, 256]))
    shape = (n1, int(rng.integers(5, 38)) * 8, int(rng.integers(5, 25)) * 8)
    u = np.asfortranarray(rng.standard_normal(shape))
    t = dev(u)
    for mu in (1, 2, 3):
        n = shape[mu - 1]
        m = int(rng.integers(n // 2, n + 40))
        mat = rng.standard_normal((m, n))
        if seed % 3 == 2:
            mat = mat + 1j * rng.standard_normal((m, n))
        a, b = policies(lambda: dv.to_host(km.mu_mode_product(t, mat, mu)))
        want = orc.mu_mode_product(u, mat, mu)
        assert orc.rel_l2(a, want) <= 1e-13, (shape, mu, m)
        assert orc.rel_l2(b, want) <= 1e-13, (shape, mu, m)
        assert orc.rel_l2(a, b) <= 1e-14, (shape, mu, m)


@pytest.mark.parametrize("policy", ["auto", "whole"])
def test_repeated_real_products_are_identical(policy):
    """A real x real k-contiguous product with half-k-block and row tails, launched many times:
    every launch must give the same, correct result (a randomised sweep once caught a
    layout / producer-warp combination that went wrong in ~1 of 10 launches)."""
    rng = np.random.default_rng(216)
    u = np.asfortranarray(rng.standard_normal((216, 213, 263)))
    mat = rng.standard_normal((194, 216)) / np.sqrt(216)
    want = orc.mu_mode_product(u, mat, 1)
    t = dev(u)
    lib = _native.lib()
    try:
        if policy == "whole":
            _native.check(lib.km_set_kernel_policy(_native.POLICY_NO_STREAMK))
        first = dv.to_host(km.mu_mode_product(t, mat, 1))
        assert orc.rel_l2(first, want) <= 1e-13
        for _ in range(60):
            assert np.array_equal(dv.to_host(km.mu_mode_product(t, mat, 1)), first)
    finally:
        _native.check(lib.km_set_kernel_policy(_native.POLICY_AUTO))
