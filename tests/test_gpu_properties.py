"""GPU: the reference's property tests (test_tensor.py:65-161, test_kron.py:116-191)
re-run against the CUDA path with hypothesis, plus edge cases (empty and extent-1
tensors, d up to 8, maximum-size state)."""

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_2103_01691_b200 as km
from oracle import kronmode_oracle as orc

pytestmark = pytest.mark.gpu

shapes = st.lists(st.integers(1, 4), min_size=1, max_size=4).map(tuple)


def loop_mu_mode(u, mat, mu):
    # Definition 1 by brute force (the reference test's oracle, test_tensor.py:10-20)
    ax = mu - 1
    out_shape = u.shape[:ax] + (mat.shape[0],) + u.shape[ax + 1:]
    out = np.zeros(out_shape, dtype=np.result_type(u.dtype, mat.dtype))
    for idx in np.ndindex(out_shape):
        acc = 0
        for j in range(u.shape[ax]):
            acc += mat[idx[ax], j] * u[idx[:ax] + (j,) + idx[ax + 1:]]
        out[idx] = acc
    return out


def kron_vec_apply(u, mats):
    big = np.ones((1, 1))
    for mat in mats:
        big = np.kron(np.asarray(mat), big)
    return big @ u.ravel(order="F")


@settings(max_examples=40, deadline=None)
@given(shape=shapes, mu=st.integers(1, 4), rows=st.integers(1, 4), seed=st.integers(0, 2**31),
       cplx=st.booleans())
def test_matches_loop_oracle(shape, mu, rows, seed, cplx):
    if mu > len(shape):
        mu = 1 + (mu - 1) % len(shape)
    rng = np.random.default_rng(seed)
    u = rng.standard_normal(shape)
    if cplx:
        u = u + 1j * rng.standard_normal(shape)
    mat = rng.standard_normal((rows, shape[mu - 1]))
    got = km.mu_mode_product(u, mat, mu)
    want = loop_mu_mode(u, mat, mu)
    assert got.dtype == want.dtype
    assert np.abs(got - want).max() <= 1e-14 * max(np.abs(want).max(), 1.0)


@settings(max_examples=30, deadline=None)
@given(shape=shapes, seed=st.integers(0, 2**31))
def test_distinct_directions_commute(shape, seed):
    if len(shape) < 2:
        shape = shape + (2,)
    rng = np.random.default_rng(seed)
    u = rng.standard_normal(shape)
    u /= np.linalg.norm(u.ravel()) or 1.0
    mu, nu = 1, len(shape)
    a = rng.standard_normal((shape[mu - 1],) * 2)
    b = rng.standard_normal((shape[nu - 1],) * 2)
    a /= np.linalg.norm(a) or 1.0
    b /= np.linalg.norm(b) or 1.0
    left = km.mu_mode_product(km.mu_mode_product(u, a, mu), b, nu)
    right = km.mu_mode_product(km.mu_mode_product(u, b, nu), a, mu)
    denom = np.linalg.norm(left.ravel()) or 1.0
    assert np.linalg.norm((left - right).ravel()) / denom <= 1e-13


@settings(max_examples=25, deadline=None)
@given(shape=st.lists(st.integers(1, 4), min_size=1, max_size=3).map(tuple), seed=st.integers(0, 2**31))
def test_kron_vec_identity(shape, seed):
    rng = np.random.default_rng(seed)
    u = rng.standard_normal(shape)
    mats = [rng.standard_normal((n, n)) for n in shape]
    got = km.tucker(u, mats).ravel(order="F")
    want = kron_vec_apply(u, mats)
    assert np.linalg.norm(got - want) / (np.linalg.norm(want) or 1.0) <= 1e-13


@pytest.mark.parametrize("d", [5, 6, 8, 9])
def test_high_order_tensors(d):
    rng = np.random.default_rng(d)
    shape = tuple(int(x) for x in rng.integers(2, 4, size=d))
    u = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    mats = [rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)) for n in shape]
    got = km.tucker(u, mats)
    assert orc.rel_l2(got, orc.tucker(u, mats)) <= 1e-13


def test_empty_and_unit_extents():
    u = np.zeros((3, 0, 2))
    got = km.mu_mode_product(u, np.ones((4, 3)), 1)
    assert got.shape == (4, 0, 2)
    v = np.arange(6.0).reshape(1, 6, 1)
    got = km.mu_mode_product(v, np.array([[2.0]]), 1)
    assert np.array_equal(got, 2 * v)
    w = np.ones((5, 1))
    got = km.mu_mode_product(w, np.ones((3, 1)), 2)
    assert got.shape == (5, 3) and np.array_equal(got, np.ones((5, 3)))


def test_zero_rows_factor():
    got = km.mu_mode_product(np.ones((3, 4)), np.ones((0, 4)), 2)
    assert got.shape == (3, 0)


def test_nonfinite_propagates_like_numpy():
    u = np.ones((4, 4))
    u[1, 2] = np.nan
    got = km.mu_mode_product(u, np.eye(4), 1)
    want = orc.mu_mode_product(u, np.eye(4), 1)
    assert np.array_equal(np.isnan(got), np.isnan(want))


@pytest.mark.slow
def test_max_size_512_step_vs_oracle():
    n = 512
    rng = np.random.default_rng(0)
    u = np.asfortranarray(rng.standard_normal((n,) * 3) + 1j * rng.standard_normal((n,) * 3))
    d2 = km.heat_factors(n, 2).factors[0]
    cache = km.prepare(km.KroneckerOp((1j * d2,) * 3), 0.01)
    got = km.step(cache, u)
    assert orc.rel_l2(got, orc.step(cache.exps, u)) <= 1e-12
