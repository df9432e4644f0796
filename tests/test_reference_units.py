"""The reference's unit tests for the hot path, run against this package.

Mirrors /root/reference/pkg/tests/test_tensor.py, test_kron.py and
test_hermite.py: same seeds, inputs and tolerances.  Tests that compute go
through the device and carry the ``gpu`` mark; the host-side builders
(Hermite basis, operators, KroneckerOp validation) run anywhere.
"""

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_2103_01691_b200 as km
from paper_2103_01691_b200.errors import (
    ConfigurationError,
    InvalidDirectionError,
    InvalidPotentialError,
    OracleSizeError,
    ShapeError,
)

gpu = pytest.mark.gpu


def loop_mu_mode(u, mat, mu):
    """Index-formula evaluation of the mode product (test_tensor.py:10-20)."""
    ax = mu - 1
    out_shape = u.shape[:ax] + (mat.shape[0],) + u.shape[ax + 1:]
    out = np.zeros(out_shape, dtype=np.result_type(u.dtype, mat.dtype))
    for idx in np.ndindex(out_shape):
        out[idx] = sum(mat[idx[ax], j] * u[idx[:ax] + (j,) + idx[ax + 1:]] for j in range(u.shape[ax]))
    return out


def kron_vec_apply(u, mats):
    big = np.ones((1, 1))
    for mat in mats:
        big = np.kron(np.asarray(mat), big)
    return big @ u.ravel(order="F")


def random_op(rng, dims, complex_factors=False):
    fs = []
    for m in dims:
        a = rng.standard_normal((m, m))
        if complex_factors:
            a = a + 1j * rng.standard_normal((m, m))
        fs.append(a)
    return km.KroneckerOp(tuple(fs))


shapes = st.lists(st.integers(1, 4), min_size=1, max_size=4).map(tuple)


# --------------------------------------------------------------- test_tensor.py


class TestMuFiberCount:
    def test_examples(self):
        assert km.mu_fiber_count((2, 3, 4), 2) == 8
        assert km.mu_fiber_count((5,), 1) == 1
        assert km.mu_fiber_count((40, 40, 40), 3) == 1600

    def test_errors(self):
        for mu in (0, 3):
            with pytest.raises(InvalidDirectionError):
                km.mu_fiber_count((2, 3), mu)
        with pytest.raises(ShapeError):
            km.mu_fiber_count((2, 0), 1)


@gpu
class TestMuModeProduct:
    def test_identity_is_bitwise_identity(self):
        u = np.asfortranarray(np.random.default_rng(7).random((3, 4, 2)) + 0.5)
        for mu in (1, 2, 3):
            assert np.array_equal(km.mu_mode_product(u, np.eye(u.shape[mu - 1]), mu), u)

    def test_row_permutation(self):
        got = km.mu_mode_product(np.array([[1.0, 2.0], [3.0, 4.0]]), np.array([[0.0, 1.0], [1.0, 0.0]]), 1)
        assert np.array_equal(got, np.array([[3.0, 4.0], [1.0, 2.0]]))

    def test_small_random_vs_loop_oracle(self):
        rng = np.random.default_rng(11)
        u, mat = rng.standard_normal((2, 3, 2)), rng.standard_normal((3, 3))
        want = loop_mu_mode(u, mat, 2)
        assert np.abs(km.mu_mode_product(u, mat, 2) - want).max() <= 1e-14 * np.abs(want).max()

    @settings(max_examples=60, deadline=None)
    @given(shape=shapes, mu=st.integers(1, 4), rows=st.integers(1, 4), seed=st.integers(0, 2**31))
    def test_matches_loop_oracle(self, shape, mu, rows, seed):
        if mu > len(shape):
            mu = 1 + (mu - 1) % len(shape)
        rng = np.random.default_rng(seed)
        u, mat = rng.standard_normal(shape), rng.standard_normal((rows, shape[mu - 1]))
        want = loop_mu_mode(u, mat, mu)
        assert np.abs(km.mu_mode_product(u, mat, mu) - want).max() <= 1e-14 * max(np.abs(want).max(), 1.0)

    @settings(max_examples=40, deadline=None)
    @given(shape=shapes, seed=st.integers(0, 2**31))
    def test_distinct_directions_commute(self, shape, seed):
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
        assert np.linalg.norm((left - right).ravel()) / (np.linalg.norm(left.ravel()) or 1.0) <= 1e-13

    def test_complex_promotion(self):
        rng = np.random.default_rng(3)
        u = rng.standard_normal((2, 3))
        mat = rng.standard_normal((3, 3)) + 1j * rng.standard_normal((3, 3))
        got = km.mu_mode_product(u, mat, 2)
        assert got.dtype == np.complex128
        assert np.abs(got - loop_mu_mode(u, mat, 2)).max() <= 1e-14

    def test_single_precision_preserved(self):
        rng = np.random.default_rng(5)
        u = rng.standard_normal((4, 4)).astype(np.float32)
        assert km.mu_mode_product(u, rng.standard_normal((4, 4)).astype(np.float32), 1).dtype == np.float32


class TestMuModeValidation:
    def test_dimension_mismatch(self):
        with pytest.raises(ShapeError):
            km.mu_mode_product(np.zeros((2, 3)), np.zeros((3, 4)), 1)

    def test_direction_out_of_range(self):
        with pytest.raises(InvalidDirectionError):
            km.mu_mode_product(np.zeros((2, 3)), np.zeros((2, 2)), 3)

    def test_tucker_error_names_direction(self):
        with pytest.raises(ShapeError, match="direction 2"):
            km.tucker(np.zeros((2, 3)), [np.eye(2), np.eye(2)])

    def test_tucker_wrong_slot_count(self):
        with pytest.raises(ShapeError):
            km.tucker(np.zeros((2, 3)), [np.eye(2)])


@gpu
class TestTucker:
    def test_all_slots_absent(self):
        u = np.arange(6.0).reshape(2, 3)
        assert np.array_equal(km.tucker(u, [None, None]), u)

    def test_two_dimensional_matrix_identity(self):
        rng = np.random.default_rng(2)
        u, l1, l2 = rng.standard_normal((3, 4)), rng.standard_normal((2, 3)), rng.standard_normal((5, 4))
        assert np.abs(km.tucker(u, [l1, l2]) - l1 @ u @ l2.T).max() <= 1e-13

    def test_matches_kron_vec_oracle(self):
        rng = np.random.default_rng(9)
        u = rng.standard_normal((3, 3, 3))
        mats = [rng.standard_normal((3, 3)) for _ in range(3)]
        want = kron_vec_apply(u, mats)
        assert np.linalg.norm(km.tucker(u, mats).ravel(order="F") - want) <= 1e-13 * np.linalg.norm(want)

    @settings(max_examples=30, deadline=None)
    @given(shape=st.lists(st.integers(1, 4), min_size=1, max_size=3).map(tuple), seed=st.integers(0, 2**31))
    def test_kron_vec_identity_small(self, shape, seed):
        rng = np.random.default_rng(seed)
        u = rng.standard_normal(shape)
        mats = [rng.standard_normal((n, n)) for n in shape]
        want = kron_vec_apply(u, mats)
        got = km.tucker(u, mats).ravel(order="F")
        assert np.linalg.norm(got - want) / (np.linalg.norm(want) or 1.0) <= 1e-13

    def test_skips_none_slots(self):
        rng = np.random.default_rng(4)
        u, mat = rng.standard_normal((2, 3, 4)), rng.standard_normal((3, 3))
        assert np.abs(km.tucker(u, [None, mat, None]) - km.mu_mode_product(u, mat, 2)).max() == 0.0


@gpu
class TestNorm:
    def test_zero_tensor(self):
        z = np.zeros((2, 2))
        assert km.norm(z, "max") == 0.0 and km.norm(z, "two") == 0.0
        assert km.norm(z, "weighted_two", weights=[np.ones(2), np.ones(2)]) == 0.0

    def test_single_entry(self):
        assert km.norm(np.array([3.0]), "max") == 3.0 and km.norm(np.array([3.0]), "two") == 3.0

    def test_weighted_example(self):
        w = [np.array([0.5, 0.5]), np.array([0.5, 0.5])]
        assert km.norm(np.ones((2, 2)), "weighted_two", weights=w) == pytest.approx(1.0, abs=1e-15)

    def test_weighted_matches_direct_sum(self):
        rng = np.random.default_rng(12)
        u = rng.standard_normal((3, 4)) + 1j * rng.standard_normal((3, 4))
        w1, w2 = rng.random(3) + 0.1, rng.random(4) + 0.1
        want = np.sqrt(sum(w1[i] * w2[j] * abs(u[i, j]) ** 2 for i in range(3) for j in range(4)))
        assert km.norm(u, "weighted_two", weights=[w1, w2]) == pytest.approx(want, rel=1e-13)


class TestNormValidation:
    def test_weight_length_mismatch(self):
        with pytest.raises(ShapeError):
            km.norm(np.ones((2, 2)), "weighted_two", weights=[np.ones(2), np.ones(3)])

    def test_unknown_kind(self):
        with pytest.raises(ConfigurationError):
            km.norm(np.ones(2), "median")


@gpu
def test_flop_counter_counts_multiply_adds():
    rng = np.random.default_rng(1)
    u, mat = rng.standard_normal((2, 3, 4)), rng.standard_normal((5, 3))
    with km.count_flops() as fc:
        km.mu_mode_product(u, mat, 2)
    assert fc.macs == 5 * 3 * 8
    km.mu_mode_product(u, mat, 2)
    assert fc.macs == 5 * 3 * 8


# ----------------------------------------------------------------- test_kron.py


class TestKroneckerOp:
    def test_shape_and_size(self):
        op = km.KroneckerOp((np.eye(2), np.eye(3), np.eye(4)))
        assert (op.shape, op.size, op.d) == ((2, 3, 4), 24, 3)

    def test_rejects(self):
        with pytest.raises(ShapeError):
            km.KroneckerOp((np.zeros((2, 3)),))
        with pytest.raises(ShapeError):
            km.KroneckerOp(())

    def test_assemble_full(self):
        a = np.random.default_rng(0).standard_normal((4, 4))
        assert np.array_equal(km.assemble_full(km.KroneckerOp((a,))), a)
        assert np.array_equal(km.assemble_full(km.KroneckerOp((np.zeros((1, 1)),) * 2)), np.zeros((1, 1)))
        op = km.KroneckerOp((np.eye(8),) * 4)
        km.assemble_full(op)
        with pytest.raises(OracleSizeError):
            km.assemble_full(op, limit=4095)

    def test_prepare(self):
        rng = np.random.default_rng(4)
        op = random_op(rng, (3, 4))
        for e, m in zip(km.prepare(op, 0.0).exps, op.shape):
            assert np.array_equal(e, np.eye(m))
        lam = np.array([-1.0, 0.5, 2.0])
        assert np.allclose(np.diag(km.prepare(km.KroneckerOp((np.diag(lam),)), 0.3).exps[0]), np.exp(0.3 * lam),
                           rtol=1e-14)
        op = random_op(np.random.default_rng(5), (4, 3))
        for e, a in zip(km.prepare(op, 0.7).exps, op.factors):
            assert np.array_equal(e, km.matexp(0.7 * a))


@gpu
class TestMatvec:
    def test_consistent_with_dense(self):
        rng = np.random.default_rng(1)
        op = random_op(rng, (2, 3))
        u = np.asfortranarray(rng.standard_normal((2, 3)))
        dense = km.assemble_full(op) @ u.ravel(order="F")
        assert np.abs(dense - km.matvec(op, u).ravel(order="F")).max() <= 1e-14 * np.abs(dense).max()

    def test_zero_factors(self):
        op = km.KroneckerOp((np.zeros((2, 2)), np.zeros((3, 3))))
        assert np.array_equal(km.matvec(op, np.ones((2, 3))), np.zeros((2, 3)))

    def test_identity_factors_give_d_times_u(self):
        u = np.random.default_rng(2).standard_normal((2, 3, 2))
        op = km.KroneckerOp(tuple(np.eye(m) for m in u.shape))
        assert np.allclose(km.matvec(op, u), 3 * u, rtol=0, atol=1e-15)

    def test_random_vs_dense_oracle(self):
        rng = np.random.default_rng(3)
        op = random_op(rng, (3, 2, 4), complex_factors=True)
        u = np.asfortranarray(rng.standard_normal((3, 2, 4)))
        want = km.assemble_full(op) @ u.ravel(order="F")
        assert np.abs(km.matvec(op, u).ravel(order="F") - want).max() <= 1e-13 * np.abs(want).max()

    def test_shape_mismatch(self):
        with pytest.raises(ShapeError):
            km.matvec(km.KroneckerOp((np.eye(2), np.eye(3))), np.ones((3, 2)))


@gpu
class TestStep:
    def test_zero_increment_is_identity(self):
        rng = np.random.default_rng(6)
        op = random_op(rng, (3, 4))
        u = np.asfortranarray(rng.standard_normal((3, 4)))
        assert np.array_equal(km.step(km.prepare(op, 0.0), u), u)

    def test_matches_dense_exponential(self):
        rng = np.random.default_rng(7)
        op = random_op(rng, (3, 3))
        u = np.asfortranarray(rng.standard_normal((3, 3)))
        got = km.step(km.prepare(op, 0.7), u).ravel(order="F")
        want = km.matexp(0.7 * km.assemble_full(op)) @ u.ravel(order="F")
        assert np.linalg.norm(got - want) <= 1e-12 * np.linalg.norm(want)

    def test_skew_hermitian_preserves_norm(self):
        rng = np.random.default_rng(8)
        fs = []
        for _ in range(3):
            b = rng.standard_normal((4, 4)) + 1j * rng.standard_normal((4, 4))
            fs.append(b - b.conj().T)
        u = np.asfortranarray(rng.standard_normal((4, 4, 4)) + 1j * rng.standard_normal((4, 4, 4)))
        v = km.step(km.prepare(km.KroneckerOp(tuple(fs)), 0.4), u)
        assert abs(km.norm(v, "two") - km.norm(u, "two")) <= 1e-13 * km.norm(u, "two")

    def test_exactness_on_random_operators(self):
        rng = np.random.default_rng(9)
        for trial in range(8):
            dims = tuple(int(rng.integers(2, 5)) for _ in range(int(rng.integers(2, 4))))
            op = random_op(rng, dims, complex_factors=bool(trial % 2))
            u = np.asfortranarray(rng.standard_normal(dims))
            tau = float(rng.uniform(0.1, 1.0))
            got = km.step(km.prepare(op, tau), u).ravel(order="F")
            want = km.matexp(tau * km.assemble_full(op)) @ u.ravel(order="F")
            assert np.linalg.norm(got - want) <= 1e-12 * np.linalg.norm(want)

    def test_semigroup_property(self):
        rng = np.random.default_rng(10)
        op = random_op(rng, (3, 4))
        u = np.asfortranarray(rng.standard_normal((3, 4)))
        one = km.step(km.prepare(op, 0.8), u)
        many, cache = u, km.prepare(op, 0.1)
        for _ in range(8):
            many = km.step(cache, many)
        assert km.norm(one - many, "two") <= 1e-11 * km.norm(one, "two")

    def test_application_order_is_immaterial(self):
        rng = np.random.default_rng(11)
        op = random_op(rng, (3, 4, 2), complex_factors=True)
        u = np.asfortranarray(rng.standard_normal((3, 4, 2)))
        cache = km.prepare(op, 0.5)
        fwd = km.step(cache, u)
        rev = u
        for mu in (3, 2, 1):
            rev = km.tucker(rev, [cache.exps[mu - 1] if m == mu else None for m in (1, 2, 3)])
        assert km.norm(fwd - rev, "two") <= 1e-12 * km.norm(fwd, "two")

    def test_constant_fixed_point_for_zero_row_sum_factors(self):
        u = np.ones((8, 8, 8), order="F")
        v = km.step(km.prepare(km.heat_factors(8, 2), 0.9), u)
        assert km.norm(v - u, "max") <= 1e-12

    def test_step_flop_count(self):
        rng = np.random.default_rng(12)
        dims = (3, 4, 5)
        op = random_op(rng, dims)
        u = np.asfortranarray(rng.standard_normal(dims))
        cache = km.prepare(op, 0.2)
        with km.count_flops() as fc:
            km.step(cache, u)
        assert fc.macs == sum(60 * m for m in dims)

    def test_shape_mismatch(self):
        with pytest.raises(ShapeError):
            km.step(km.prepare(km.KroneckerOp((np.eye(2), np.eye(3))), 0.1), np.ones((2, 4)))


# -------------------------------------------------------------- test_hermite.py


class TestHermiteHost:
    def test_eval(self):
        assert km.hermite_eval(1, 0.0)[0] == pytest.approx(np.pi**-0.25, rel=1e-15)
        assert km.hermite_eval(2, 0.0)[1] == 0.0
        assert km.hermite_eval(6, 1.3)[5] == pytest.approx(-0.39939146281375073457, rel=1e-13)
        assert km.hermite_eval(4, np.array([0.0, 1.0, 2.0])).shape == (4, 3)

    def test_gauss_hermite(self):
        nodes, weights = km.gauss_hermite(1)
        assert nodes[0] == 0.0 and weights[0] == pytest.approx(np.sqrt(np.pi), rel=1e-15)
        nodes, weights = km.gauss_hermite(2)
        assert np.allclose(nodes, [-2.0**-0.5, 2.0**-0.5], rtol=1e-14)
        nodes, _ = km.gauss_hermite(31)
        assert np.abs(nodes + nodes[::-1]).max() == 0.0
        for k in (0, 501):
            with pytest.raises(ConfigurationError):
                km.gauss_hermite(k)

    @pytest.mark.parametrize("k", [20, 64, 100])
    def test_discrete_orthonormality(self, k):
        b = km.hermite_basis(k)
        assert np.abs((b.phi * b.mod_weights) @ b.phi.T - np.eye(k)).max() <= 1e-12

    def test_harmonic_eigenvalues(self):
        assert km.harmonic_eigenvalues((4, 4, 4))[0, 0, 0] == 1.5
        assert km.harmonic_eigenvalues((8,))[5] == 5.5
        lam = km.harmonic_eigenvalues((5, 6))
        assert (np.diff(lam, axis=0) > 0).all() and (np.diff(lam, axis=1) > 0).all()

    def test_operators(self):
        x8 = km.position_operator(km.hermite_basis(8))
        assert x8[0, 1] == pytest.approx(2.0**-0.5, rel=1e-13)
        assert np.abs(np.diag(x8)).max() <= 1e-14
        x12 = km.position_operator(km.hermite_basis(12))
        assert np.abs(x12 - x12.T).max() <= 1e-14
        k = 30
        want = np.zeros((k, k))
        for i in range(k - 1):
            want[i, i + 1] = want[i + 1, i] = np.sqrt((i + 1) / 2.0)
        assert np.abs(km.position_operator(km.hermite_basis(k)) - want).max() <= 1e-12
        assert np.abs(km.potential_operator(km.hermite_basis(10), lambda x: np.ones_like(x)) - np.eye(10)).max() <= 1e-13
        b9 = km.hermite_basis(9)
        assert np.abs(km.potential_operator(b9, lambda x: x) - km.position_operator(b9)).max() <= 1e-14
        b8 = km.hermite_basis(8)
        diff = km.potential_operator(b8, lambda x: x * x, quad=16) - km.position_operator(b8) @ km.position_operator(b8)
        assert diff[-1, -1] == pytest.approx(4.0, rel=1e-12)
        diff[-1, -1] = 0.0
        assert np.abs(diff).max() <= 1e-12
        with pytest.raises(InvalidPotentialError):
            with np.errstate(divide="ignore"):
                km.potential_operator(km.hermite_basis(3), lambda x: np.where(x == 0, np.inf, x))

    def test_hamiltonian_factor(self):
        a = km.hamiltonian_factor(km.hermite_basis(10), lambda x: 0.5 * x * x)
        assert np.abs(a - (-1j * np.diag(np.arange(10) + 0.5))).max() == 0.0
        a = km.hamiltonian_factor(km.hermite_basis(16), lambda x: np.cos(2 * np.pi * x))
        assert np.abs(a + a.conj().T).max() <= 1e-12
        a = km.hamiltonian_factor(km.hermite_basis(8), lambda x: np.cos(2 * np.pi * x))
        u = km.matexp(0.7 * a)
        assert np.abs(u.conj().T @ u - np.eye(8)).max() <= 1e-12


@gpu
class TestTransforms:
    def test_ground_state_maps_to_unit_coefficient(self):
        b = km.hermite_basis(12)
        g = km.hermite_eval(1, b.nodes)[0]
        want = np.zeros((12, 12))
        want[0, 0] = 1.0
        assert np.abs(km.forward_transform((b, b), np.outer(g, g)) - want).max() <= 1e-13

    def test_zero_field(self):
        assert np.abs(km.forward_transform((km.hermite_basis(5),), np.zeros(5))).max() == 0.0

    def test_linearity_on_two_modes(self):
        b = km.hermite_basis(16)
        phi = km.hermite_eval(16, b.nodes)
        want = np.zeros(16)
        want[3], want[7] = 1.0, 2.0
        assert np.abs(km.forward_transform((b,), phi[3] + 2.0 * phi[7]) - want).max() <= 1e-12

    def test_round_trip(self):
        rng = np.random.default_rng(0)
        bases = (km.hermite_basis(32),) * 2
        v = rng.standard_normal((32, 32)) + 1j * rng.standard_normal((32, 32))
        back = km.inverse_transform(bases, km.forward_transform(bases, v))
        assert np.abs(back - v).max() <= 1e-11 * np.abs(v).max()

    def test_coefficient_space_round_trip(self):
        c = np.random.default_rng(1).standard_normal((16, 16, 16))
        bases = (km.hermite_basis(16),) * 3
        again = km.forward_transform(bases, km.inverse_transform(bases, c))
        assert np.abs(again - c).max() <= 1e-11 * np.abs(c).max()

    def test_unit_coefficient_reconstructs_ground_state(self):
        b = km.hermite_basis(6)
        f = np.zeros((6, 6))
        f[0, 0] = 1.0
        assert np.abs(km.inverse_transform((b, b), f) - np.outer(b.phi[0], b.phi[0])).max() <= 1e-14

    def test_evaluation_at_arbitrary_points(self):
        c = np.random.default_rng(2).standard_normal(10)
        b = km.hermite_basis(10)
        got = km.inverse_transform((b,), c, eval_points=[np.array([0.0])])
        want = sum(c[i] * km.hermite_eval(10, 0.0)[i] for i in range(10))
        assert got[0] == pytest.approx(want, rel=1e-13)

    def test_parseval(self):
        rng = np.random.default_rng(3)
        b = km.hermite_basis(20)
        v = rng.standard_normal((20, 20)) + 1j * rng.standard_normal((20, 20))
        c = km.forward_transform((b, b), v)
        weighted = km.norm(v, "weighted_two", weights=[b.mod_weights] * 2)
        assert abs(weighted - km.norm(c, "two")) <= 1e-12 * weighted


class TestTransformValidation:
    def test_shape_validation(self):
        b = km.hermite_basis(4)
        with pytest.raises(ShapeError):
            km.forward_transform((b,), np.zeros(5))
        with pytest.raises(ShapeError):
            km.inverse_transform((b,), np.zeros(4), eval_points=[np.zeros(3), np.zeros(3)])
