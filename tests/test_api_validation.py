"""CPU: argument validation of the drop-in API raises the reference's
exception classes and messages before any device work
(tensor.py:62-66, 102-111, 151-161; kron.py:23-48, 119-120; hermite.py:102-105;
problems.py:528-539, 556-557)."""

import numpy as np
import pytest

import paper_2103_01691_b200 as km
from paper_2103_01691_b200 import ConfigurationError, InvalidDirectionError, ShapeError
from paper_2103_01691_b200.tensor import count_flops, mu_fiber_count


class TestMuFiberCount:
    def test_examples(self):
        assert mu_fiber_count((2, 3, 4), 2) == 8
        assert mu_fiber_count((5,), 1) == 1
        assert mu_fiber_count((40, 40, 40), 3) == 1600

    def test_errors(self):
        with pytest.raises(InvalidDirectionError):
            mu_fiber_count((2, 3), 0)
        with pytest.raises(InvalidDirectionError):
            mu_fiber_count((2, 3), 3)
        with pytest.raises(ShapeError):
            mu_fiber_count((2, 0), 1)


def test_mu_mode_dimension_mismatch():
    with pytest.raises(ShapeError, match="direction 1: matrix has 4 columns, tensor extent is 2"):
        km.mu_mode_product(np.zeros((2, 3)), np.zeros((3, 4)), 1)


def test_mu_mode_direction_out_of_range():
    with pytest.raises(InvalidDirectionError, match="direction 3 outside 1..2"):
        km.mu_mode_product(np.zeros((2, 3)), np.zeros((2, 2)), 3)
    with pytest.raises(InvalidDirectionError, match="must be an integer"):
        km.mu_mode_product(np.zeros((2, 3)), np.zeros((2, 2)), 1.0)


def test_mu_mode_operator_not_matrix():
    with pytest.raises(ShapeError, match="must be a matrix"):
        km.mu_mode_product(np.zeros((2, 3)), np.zeros(2), 1)


def test_tucker_error_names_direction():
    with pytest.raises(ShapeError, match="direction 2"):
        km.tucker(np.zeros((2, 3)), [np.eye(2), np.eye(2)])


def test_tucker_wrong_slot_count():
    with pytest.raises(ShapeError):
        km.tucker(np.zeros((2, 3)), [np.eye(2)])


def test_tucker_all_absent_is_identity():
    u = np.arange(6.0).reshape(2, 3)
    assert np.array_equal(km.tucker(u, [None, None]), u)


def test_step_shape_mismatch():
    cache = km.prepare(km.KroneckerOp((np.eye(2), np.eye(3))), 0.1)
    with pytest.raises(ShapeError):
        km.step(cache, np.ones((2, 4)))


def test_kronecker_op_validation():
    with pytest.raises(ShapeError):
        km.KroneckerOp((np.zeros((2, 3)),))
    with pytest.raises(ShapeError):
        km.KroneckerOp(())
    op = km.KroneckerOp((np.eye(2), np.eye(3), np.eye(4)))
    assert op.shape == (2, 3, 4) and op.size == 24 and op.d == 3


def test_prepare_zero_is_identity_on_host():
    cache = km.prepare(km.KroneckerOp((np.ones((3, 3)), np.ones((4, 4)))), 0.0)
    for e, m in zip(cache.exps, (3, 4)):
        assert np.array_equal(e, np.eye(m))


def test_flop_counter_counts_before_device():
    # the tally happens in the host mirror; without a GPU the call then fails
    u = np.ones((2, 3, 4))
    with count_flops() as fc:
        try:
            km.mu_mode_product(u, np.ones((5, 3)), 2)
        except km.DeviceError:
            pass
    assert fc.macs == 5 * 3 * 8


def test_norm_validation():
    with pytest.raises(ConfigurationError):
        km.norm(np.ones(2), "median")
    with pytest.raises(ShapeError):
        km.norm(np.ones((2, 2)), "weighted_two", weights=[np.ones(2), np.ones(3)])
    with pytest.raises(ConfigurationError):
        km.norm(np.ones((2, 2)), "weighted_two")


def test_hermite_shape_validation():
    basis = km.hermite_basis(4)
    with pytest.raises(ShapeError):
        km.forward_transform((basis,), np.zeros(5))
    with pytest.raises(ShapeError):
        km.inverse_transform((basis,), np.zeros(4), eval_points=[np.zeros(3), np.zeros(3)])


def test_gpe_step_validation():
    grids, lin_op, weights = km.gpe_setup(16)
    cache = km.prepare(lin_op, 0.0)
    with pytest.raises(ShapeError):
        km.gpe_strang_step(cache, weights, np.ones((4, 4, 4), complex), 0.1)
    with pytest.raises(ShapeError, match="direction 2: weight vector"):
        km.gpe_strang_step(cache, [weights[0], weights[1][:3], weights[2]],
                           np.ones((16, 16, 16), complex), 0.1)
