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
