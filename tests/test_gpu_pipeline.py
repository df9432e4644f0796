"""GPU: the host-pipelined path (numpy in/out >= 16 MB, _pipeline.py) against the oracle.
Covers slabs with pre/post phases, skipped last direction, rectangular factors,
dtype promotion and page-locked inputs."""

import numpy as np
import pytest

import paper_2103_01691_b200 as km
from oracle import kronmode_oracle as orc
from paper_2103_01691_b200 import _pipeline

pytestmark = pytest.mark.gpu

N = 128


def crand(rng, shape):
    return np.asfortranarray(rng.standard_normal(shape) + 1j * rng.standard_normal(shape))


def schrod(n, tau=0.01):
    d2 = km.heat_factors(n, 2).factors[0]
    return km.prepare(km.KroneckerOp((1j * d2,) * 3), tau)


def test_pipeline_is_taken_for_large_host_inputs():
    assert _pipeline.eligible(np.empty((N, N, N), complex), 3)
    assert not _pipeline.eligible(np.empty((16, 16, 16), complex), 3)


def test_step_pipelined_vs_oracle():
    rng = np.random.default_rng(0)
    u = crand(rng, (N, N, N))
    cache = schrod(N)
    assert orc.rel_l2(km.step(cache, u), orc.step(cache.exps, u)) <= 1e-12


def test_step_pinned_input():
    import torch

    rng = np.random.default_rng(1)
    u = crand(rng, (N, N, N))
    buf = torch.empty((N, N, N), dtype=torch.complex128, pin_memory=True).numpy()
    buf[...] = u.transpose(2, 1, 0)
    host = buf.transpose(2, 1, 0)
    cache = schrod(N)
    got = km.step(cache, host)
    assert got.flags.f_contiguous
    assert orc.rel_l2(got, orc.step(cache.exps, u)) <= 1e-12


def test_tucker_skip_last_direction_and_rectangular():
    rng = np.random.default_rng(2)
    u = crand(rng, (N, N, N))
    a = rng.standard_normal((96, N)) + 1j * rng.standard_normal((96, N))
    b = rng.standard_normal((160, N))
    got = km.tucker(u, [a, b, None])
    assert got.shape == (96, 160, N)
    assert orc.rel_l2(got, orc.tucker(u, [a, b, None])) <= 1e-12
    c = rng.standard_normal((40, N))
    got2 = km.tucker(u, [None, None, c])
    assert orc.rel_l2(got2, orc.tucker(u, [None, None, c])) <= 1e-12


def test_real_input_complex_factors():
    rng = np.random.default_rng(3)
    u = np.asfortranarray(rng.standard_normal((N, N, N)))
    cache = schrod(N)
    got = km.step(cache, u)
    assert got.dtype == np.complex128
    assert orc.rel_l2(got, orc.step(cache.exps, u)) <= 1e-12


def test_gpe_strang_pipelined_vs_oracle():
    grids, lin_op, weights = km.gpe_setup(N)
    from paper_2103_01691_b200.problems import weighted_vortex_state

    psi = weighted_vortex_state(grids, weights)
    cache = km.prepare(lin_op, 0.1)
    got = km.gpe_strang_step(cache, weights, psi, 0.1)
    want = orc.gpe_strang_step(cache.exps, weights, psi, 0.1)
    assert orc.rel_l2(got, want) <= 1e-12


def test_tdpot_pipelined_vs_oracle():
    from paper_2103_01691_b200.hermite import physical_propagator
    from paper_2103_01691_b200.problems import schrodinger_initial_state

    b = km.hermite_basis(N)
    p = physical_propagator(b, 0.02)
    cache = km.PropagatorCache(0.02, (p, p, p))
    psi = schrodinger_initial_state((b.nodes,) * 3)
    got = km.tdpot_strang_step(cache, b.nodes, psi, 0.3, 0.02)
    want = orc.tdpot_strang_step(cache.exps, b.nodes, psi, 0.3, 0.02)
    assert orc.rel_l2(got, want) <= 1e-12


def test_hermite_transforms_pipelined():
    b = km.hermite_basis(N)
    rng = np.random.default_rng(4)
    vals = crand(rng, (N, N, N))
    fwd = km.forward_transform((b,) * 3, vals)
    want = orc.forward_transform([b.phi] * 3, [b.mod_weights] * 3, vals)
    assert orc.rel_l2(fwd, want) <= 1e-12
    back = km.inverse_transform((b,) * 3, fwd)
    assert orc.rel_l2(back, vals) <= 1e-11


@pytest.mark.parametrize("cplx", [True, False])
def test_mumode_fibers_matches_the_full_product(cplx):
    """km_mumode_fibers (the first output row block in fiber pieces) writes exactly the
    requested fibers of the trailing-direction product, bit for bit, and nothing else."""
    import ctypes

    import torch

    from paper_2103_01691_b200 import _device as dv, _native

    rng = np.random.default_rng(5)
    shape, m = (64, 48, 40), 24
    u = crand(rng, shape) if cplx else np.asfortranarray(rng.standard_normal(shape))
    mat = rng.standard_normal((m, shape[2])) + (1j * rng.standard_normal((m, shape[2])) if cplx else 0)
    dev = torch.device("cuda", 0)
    code = _native.KM_C128 if cplx else _native.KM_F64
    t = dv.to_device(u, u.dtype, dev)
    L = torch.from_numpy(np.ascontiguousarray(mat)).to(dev)  # row-major, as the ABI takes factors
    full = dv.to_host(km.mu_mode_product(t, L, 3)).reshape(-1, m, order="F")
    nl = shape[0] * shape[1]
    lib = _native.lib()
    for f0, nf in [(0, nl), (128, 1000), (nl - 1, 1), (512, 1024)]:
        out = torch.zeros(nl * m, dtype=t.dtype, device=dev)
        _native.check(lib.km_mumode_fibers(t.data_ptr(), code, L.data_ptr(), code, out.data_ptr(), m, nl,
                                           shape[2], f0, nf, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
        got = out.cpu().numpy().reshape(nl, m, order="F")
        assert np.array_equal(got[f0:f0 + nf], full[f0:f0 + nf])
        assert not got[:f0].any() and not got[f0 + nf:].any()
    with pytest.raises(Exception):
        _native.check(lib.km_mumode_fibers(t.data_ptr(), code, L.data_ptr(), code, out.data_ptr(), m, nl,
                                           shape[2], nl - 4, 8, None))


def test_real_step_pipelined_vs_oracle():
    rng = np.random.default_rng(6)
    u = np.asfortranarray(rng.standard_normal((N, N, N)))
    d2 = km.heat_factors(N, 2).factors[0]
    cache = km.prepare(km.KroneckerOp((d2,) * 3), 1e-4)
    assert orc.rel_l2(km.step(cache, u), orc.step(cache.exps, u)) <= 1e-12
