"""The fused first-two-products launch for small 3-D complex128 planes (km_tucker's
mumode_plane12_kernel, csrc/kmb200_plane.cuh) against the oracle, against the per-product
launches (KM_POLICY_NO_PLANE_FUSION), inside the GPE Strang step (phase pre-pass and fused
post-phase on the third product), and which kernels actually ran."""

import numpy as np
import pytest

import paper_2103_01691_b200 as km
from conftest import kernels_launched
from oracle import kronmode_oracle as orc
from paper_2103_01691_b200 import _device as dv, _native

pytestmark = pytest.mark.gpu


def _policy(p):
    _native.check(_native.lib().km_set_kernel_policy(p))


def _rand(shape, seed):
    rng = np.random.default_rng(seed)
    return np.asfortranarray(rng.standard_normal(shape) + 1j * rng.standard_normal(shape))


@pytest.mark.parametrize("dims", [(64, 64, 64), (48, 48, 48), (32, 32, 32), (64, 32, 40), (32, 64, 3),
                                  (48, 64, 200), (64, 48, 1)])
def test_plane_fusion_matches_oracle_and_per_product(dims):
    import torch

    u = _rand(dims, sum(dims))
    mats = [_rand((n, n), n + 7) / n for n in dims]
    t = dv.to_device(u, np.complex128, dv.device())
    dm = [dv.matrix_to_device(m, np.complex128, t.device) for m in mats]
    try:
        _policy(_native.POLICY_AUTO)
        fused, names = kernels_launched(lambda: km.tucker(t, dm))
        _policy(_native.POLICY_NO_PLANE_FUSION)
        sep, names_sep = kernels_launched(lambda: km.tucker(t, dm))
    finally:
        _policy(_native.POLICY_AUTO)
    want = orc.tucker(u, mats)
    assert orc.rel_l2(dv.to_host(fused), want) <= 1e-13
    assert orc.rel_l2(dv.to_host(fused), dv.to_host(sep)) <= 1e-14
    if names is not None and names_sep is not None:
        assert any("mumode_plane12_kernel" in n for n in names)
        assert not any("mumode_plane12_kernel" in n for n in names_sep)
    torch.cuda.synchronize()


def test_plane_fusion_not_used_outside_its_shapes():
    """Planes above 64 x 64, rectangular first factors and real factors keep per-product launches."""
    for dims, rect in (((96, 96, 8), False), ((64, 64, 64), True)):
        u = _rand(dims, 5)
        mats = [_rand((n, n), n) / n for n in dims]
        if rect:
            mats[0] = _rand((32, dims[0]), 9) / dims[0]
        t = dv.to_device(u, np.complex128, dv.device())
        got, names = kernels_launched(lambda: km.tucker(t, [dv.matrix_to_device(m, np.complex128, t.device)
                                                            for m in mats]))
        assert orc.rel_l2(dv.to_host(got), orc.tucker(u, mats)) <= 1e-13
        if names is not None:
            assert not any("mumode_plane12_kernel" in n for n in names)


def test_plane_fusion_in_gpe_strang_step():
    """64^3 GPE step: the opening phase as km_tucker's pre-pass, products 1+2 fused, the closing
    phase in the third product's epilogue."""
    n = 64
    _, lin_op, weights = km.gpe_setup(n)
    cache = km.prepare(lin_op, 0.05)
    psi = _rand((n,) * 3, 3) * 0.1
    t = dv.to_device(psi, np.complex128, dv.device())
    got, names = kernels_launched(lambda: km.gpe_strang_step(cache, weights, t, 0.05))
    want = orc.gpe_strang_step(cache.exps, weights, psi, 0.05)
    assert orc.rel_l2(dv.to_host(got), want) <= 1e-12
    if names is not None:
        assert any("mumode_plane12_kernel" in n for n in names)


def test_plane_fusion_ten_steps_graph_replay():
    """Config 1 as the bench runs it: ten 64^3 steps captured into a CUDA graph (fused planes
    under capture), equal to ten eager per-product steps."""
    import torch

    from paper_2103_01691_b200 import dist

    n = 64
    u = _rand((n,) * 3, 11)
    d2 = km.heat_factors(n, 2).factors[0]
    cache = km.prepare(km.KroneckerOp((1j * d2,) * 3), 0.01)
    mats = cache.device_exps((np.complex128,) * 3, dv.device())
    st = dist.LocalStepper(dv.to_device(u, np.complex128, dv.device()), mats)
    assert st.launches_per_step == 2
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
        for _ in range(10):
            st.step()
    g.replay()
    torch.cuda.synchronize()
    want = u
    for _ in range(10):
        want = orc.step(cache.exps, want)
    assert orc.rel_l2(dv.to_host(st.a), want) <= 1e-12


@pytest.mark.parametrize("dims", [(64, 64, 300), (48, 32, 333)])
def test_plane_fusion_after_a_pre_pass_many_waves(dims):
    """GPE step on rectangular states with hundreds of planes (several waves of plane CTAs): the
    opening phase must land in a buffer the fused launch does not write (km_tucker puts it in
    ws1 / out, the fused launch writes ws0), otherwise a plane's CTAs would overwrite rows another
    CTA of the same plane has not loaded yet."""
    rng = np.random.default_rng(sum(dims))
    factors = []
    for n in dims:
        h = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
        factors.append(-0.5j * (h + h.conj().T) / n)
    cache = km.prepare(km.KroneckerOp(tuple(factors)), 0.1)
    weights = [0.5 + rng.random(n) for n in dims]
    psi = _rand(dims, 21) * 0.3
    t = dv.to_device(psi, np.complex128, dv.device())
    got, names = kernels_launched(lambda: km.gpe_strang_step(cache, weights, t, 0.1))
    want = orc.gpe_strang_step(cache.exps, weights, psi, 0.1)
    assert orc.rel_l2(dv.to_host(got), want) <= 1e-12
    if names is not None:
        assert any("mumode_plane12_kernel" in n for n in names)


@pytest.mark.parametrize("dims,steps", [((64, 64, 64), 10), ((64, 64, 64), 1), ((64, 64, 64), 3),
                                        ((48, 48, 48), 4), ((32, 64, 48), 5), ((64, 32, 32), 2)])
def test_steps_paired_matches_oracle_and_per_step(dims, steps):
    """km_steps_paired (LocalStepper.run): two steps per three fused launches, step s+1 in the
    direction order 3, 1, 2 -- equal to the step-by-step oracle up to rounding."""
    from paper_2103_01691_b200 import dist

    u = _rand(dims, sum(dims) + steps)
    factors = []
    rng = np.random.default_rng(steps)
    for n in dims:
        h = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
        factors.append(-0.5j * (h + h.conj().T) / n)
    cache = km.prepare(km.KroneckerOp(tuple(factors)), 0.2)
    mats = cache.device_exps((np.complex128,) * 3, dv.device())
    st = dist.LocalStepper(dv.to_device(u, np.complex128, dv.device()), mats)
    assert st.paired_ok() and st.launches_for(steps) == (steps // 2) * 3 + (steps % 2) * 2
    _, names = kernels_launched(lambda: st.run(steps))
    ref = dist.LocalStepper(dv.to_device(u, np.complex128, dv.device()), mats)
    ref.run(steps, paired=False)
    want = u
    for _ in range(steps):
        want = orc.step(cache.exps, want)
    got = dv.to_host(st.a)
    assert orc.rel_l2(got, want) <= 1e-13
    assert orc.rel_l2(got, dv.to_host(ref.a)) <= 1e-14
    if names is not None and any("mumode_" in n for n in names):
        # (CUPTI may drop records late in a long test process: require the fused launches only
        # when it delivered the step's other launches)
        fused = any("mumode_plane12_kernel" in n or "mumode_pencil33_kernel" in n for n in names)
        assert fused, names


def test_steps_paired_graph_and_abi_errors():
    import ctypes

    import torch

    from paper_2103_01691_b200 import dist

    n = 64
    u = _rand((n,) * 3, 31)
    d2 = km.heat_factors(n, 2).factors[0]
    cache = km.prepare(km.KroneckerOp((1j * d2,) * 3), 0.01)
    mats = cache.device_exps((np.complex128,) * 3, dv.device())
    st = dist.LocalStepper(dv.to_device(u, np.complex128, dv.device()), mats)
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
        st.run(10)
    g.replay()
    torch.cuda.synchronize()
    want = u
    for _ in range(10):
        want = orc.step(cache.exps, want)
    assert orc.rel_l2(dv.to_host(st.a), want) <= 1e-12
    lib = _native.lib()
    a, b, w = st.a, st.b, st.w
    p = [ctypes.c_void_p(m.data_ptr()) for m in mats]
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    assert lib.km_steps_paired(a.data_ptr(), *p, n, n, n, 2, a.data_ptr(), w.data_ptr(), stream) == _native.KM_EINVAL
    assert lib.km_steps_paired(a.data_ptr(), *p, n, n, 96, 2, b.data_ptr(), w.data_ptr(), stream) == _native.KM_EINVAL
    assert lib.km_steps_paired(a.data_ptr(), *p, n, n, n, 0, b.data_ptr(), w.data_ptr(), stream) == _native.KM_EINVAL
