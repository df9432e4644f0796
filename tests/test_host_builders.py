"""Host-side builders (grids, stencils, boundary conditions, dense helpers) against
the checks of the reference's test_fd.py and test_linalg.py.

These run on the CPU: they are the inputs of the hot path, not the hot path.
The few checks that apply an operator (``matvec``) go through the device and
carry the ``gpu`` mark.
"""

import numpy as np
import pytest

import paper_2103_01691_b200 as km
from paper_2103_01691_b200 import fd
from paper_2103_01691_b200.errors import (ConfigurationError, InvalidGridError, InvalidInputError, ShapeError,
                                          SingularMatrixError)


# ------------------------------------------------------------------ stencils (test_fd.py:30-97)


def test_fd_weights_known_stencils():
    h = 0.25
    assert np.allclose(fd.fd_weights([-h, 0.0, h], 0.0, 2), np.array([1.0, -2.0, 1.0]) / h**2, rtol=1e-13)
    h = 0.5
    w = fd.fd_weights(h * np.arange(-2.0, 3.0), 0.0, 2)
    assert np.allclose(w, np.array([-1 / 12, 4 / 3, -5 / 2, 4 / 3, -1 / 12]) / h**2, rtol=1e-12)
    assert np.allclose(fd.fd_weights([0.0, 0.1], 0.0, 1), [-10.0, 10.0], rtol=1e-13)
    w0 = fd.fd_weights([-1.0, 0.5, 2.0], 0.3, 0)  # interpolation
    assert w0 @ np.array([1.0, 0.25, 4.0]) == pytest.approx(0.09, rel=1e-12)


@pytest.mark.parametrize("seed", range(8))
def test_fd_weights_polynomial_exactness(seed):
    rng = np.random.default_rng(seed)
    nodes = np.cumsum(0.2 + rng.random(6))
    center = float(rng.uniform(nodes[0], nodes[-1]))
    for deriv in range(4):
        w = fd.fd_weights(nodes, center, deriv)
        for degree in range(6):
            coeffs = np.zeros(degree + 1)
            coeffs[0] = 1.0
            want = np.polyval(np.polyder(coeffs, deriv), center) if deriv <= degree else 0.0
            assert w @ np.polyval(coeffs, nodes) == pytest.approx(want, abs=1e-8 * max(np.abs(w).max(), 1.0))


def test_fd_weights_errors():
    with pytest.raises(InvalidGridError):
        fd.fd_weights([0.0, 0.0, 1.0], 0.0, 1)
    with pytest.raises(ConfigurationError):
        fd.fd_weights([0.0, 1.0], 0.0, 2)


# ------------------------------------------------------------ diff matrices (test_fd.py:100-165)


def test_diff_matrix_closures():
    d2 = fd.diff_matrix(fd.uniform_periodic_grid(0.0, 4.0, 4), 2, 2, fd.PERIODIC_BC)
    for i in range(4):
        assert np.allclose(d2[i], np.roll([-2.0, 1.0, 0.0, 1.0], i), rtol=0, atol=1e-14)
    d2 = fd.diff_matrix(fd.uniform_grid(0.0, 1.0, 3), 2, 2, fd.DIRICHLET_BC)
    assert np.allclose(d2, np.array([[-2.0, 1, 0], [1, -2, 1], [0, 1, -2]]) / 0.25, rtol=0, atol=1e-12)
    d1 = fd.diff_matrix(fd.uniform_grid(0.0, 1.0, 9), 1, 2, fd.NEUMANN_BC)
    assert np.abs(d1[0]).max() == 0.0 and np.abs(d1[-1]).max() == 0.0
    for g in (fd.uniform_grid(0.0, 1.0, 7), fd.nonuniform_grid([0.0, 0.1, 0.35, 0.6, 1.0])):
        assert np.abs(fd.diff_matrix(g, 2, 2, fd.NEUMANN_BC) @ np.ones(g.n)).max() <= 1e-8


def test_diff_matrix_nonuniform_exactness_and_pairs():
    g = fd.nonuniform_grid([0.0, 0.3, 0.7, 1.4, 2.0])
    d2 = fd.diff_matrix(g, 2, 2, fd.NEUMANN_BC)
    assert np.allclose((d2 @ g.points**2)[1:-1], 2.0, atol=1e-10)
    # a plain (left, right) pair is accepted as well as a BoundaryCondition
    assert np.array_equal(d2, fd.diff_matrix(g, 2, 2, ("neumann_zero", "neumann_zero")))


def test_diff_matrix_order_four_interior():
    g = fd.uniform_grid(0.0, 2.0, 12)
    d1, d2 = (fd.diff_matrix(g, k, 4, fd.DIRICHLET_BC) for k in (1, 2))
    x = g.points
    tol = 100 * np.finfo(float).eps * max(np.abs(d2).max(), 1.0)
    for deg in range(5):
        dy = deg * x ** max(deg - 1, 0) if deg else 0 * x
        ddy = deg * (deg - 1) * x ** max(deg - 2, 0) if deg >= 2 else 0 * x
        assert np.abs((d2 @ x**deg - ddy)[2:-2]).max() <= tol
        assert np.abs((d1 @ x**deg - dy)[2:-2]).max() <= tol


def test_periodic_eigenvalues():
    for n in (6, 10, 16):
        g = fd.uniform_periodic_grid(0.0, 2 * np.pi, n)
        got = np.sort(np.linalg.eigvalsh(fd.diff_matrix(g, 2, 2, fd.PERIODIC_BC)))
        want = np.sort((2 * np.cos(2 * np.pi * np.arange(n) / n) - 2) / g.spacing**2)
        assert np.abs(got - want).max() <= 1e-10 / g.spacing**2


def test_diff_matrix_and_bc_errors():
    g = fd.uniform_grid(0.0, 1.0, 5)
    for args in ((g, 3, 2, fd.DIRICHLET_BC), (g, 2, 3, fd.DIRICHLET_BC), (g, 2, 6, fd.DIRICHLET_BC),
                 (g, 2, 2, fd.PERIODIC_BC), (fd.nonuniform_grid([0.0, 0.1, 0.4, 0.5, 1.0]), 2, 4, fd.NEUMANN_BC)):
        with pytest.raises(ConfigurationError):
            fd.diff_matrix(*args)
    with pytest.raises(ConfigurationError):
        fd.BoundaryCondition("periodic", "dirichlet_zero")
    with pytest.raises(ConfigurationError):
        fd.BoundaryCondition("clamped", "clamped")
    assert fd.PERIODIC_BC.is_periodic and not fd.NEUMANN_BC.is_periodic


# ------------------------------------------------------------------------ grids (test_fd.py:168-190)


def test_grids():
    with pytest.raises(InvalidGridError):
        fd.nonuniform_grid([0.0, 0.5, 0.5, 1.0])
    g = fd.uniform_periodic_grid(0.0, 2 * np.pi, 8)
    assert g.n == 8 and g.points[0] == 0.0 and g.points[-1] < 2 * np.pi
    assert g.spacing == pytest.approx(np.pi / 4)
    s = fd.sinh_clustered_grid(17, half_width=20.0, strength=2.0)
    assert s.points[0] == pytest.approx(-20.0) and s.points[-1] == pytest.approx(20.0)
    gaps = np.diff(s.points)
    assert gaps.min() == gaps[len(gaps) // 2]
    with pytest.raises(ConfigurationError):
        s.spacing
    with pytest.raises(ConfigurationError):
        fd.Grid1D(np.arange(3.0), "staggered")


# --------------------------------------------------------- model factors (test_fd.py:193-281)


def test_heat_factors():
    h = 2 * np.pi / 40
    eigs = np.linalg.eigvalsh(fd.heat_factors(40, 2).factors[0])
    assert eigs.min() >= -4.0 / h**2 * (1 + 1e-12) and eigs.max() <= 1e-10
    x = 2 * np.pi * np.arange(8) / 8
    assert np.abs(fd.heat_factors(8, np.inf).factors[0] @ np.cos(x) + np.cos(x)).max() <= 1e-12
    with pytest.raises(ConfigurationError):
        fd.heat_factors(16, 3)
    with pytest.raises(ConfigurationError):
        fd.fourier_second_derivative(9)


def test_pipeflow_factors():
    assert 1.9999 < fd.pipeflow_velocity(0.0) < 2.0001
    assert fd.pipeflow_velocity(15.0 / 4.0) == pytest.approx(4.0, abs=2e-2)
    _, z = fd.pipeflow_grids(16)
    d1 = fd.diff_matrix(z, 1, 2, fd.BoundaryCondition(fd.DIRICHLET_ZERO, fd.NEUMANN_ZERO))
    assert np.abs((d1 @ np.ones(16))[1:-1]).max() <= 1e-12
    with pytest.raises(ConfigurationError):
        fd.pipeflow_factors(4)


def test_gpe_factors():
    g = fd.uniform_grid(-1.0, 1.0, 10)
    raw = 0.5 * fd.diff_matrix(g, 2, 2, fd.NEUMANN_BC)
    op, w = fd.gpe_weighted_factors([g])
    assert np.abs(op.factors[0][2:-2, 2:-2] - raw[2:-2, 2:-2]).max() <= 1e-13
    assert w[0][1] == pytest.approx(g.spacing)
    a = fd.gpe_weighted_factors([fd.nonuniform_grid([-2.0, -1.1, -0.3, 0.4, 1.2, 2.0])])[0].factors[0]
    assert np.abs(a - a.T).max() <= 1e-10
    s = fd.sinh_clustered_grid(32)
    got = np.sort(np.linalg.eigvalsh(fd.gpe_weighted_factors([s])[0].factors[0]))
    want = np.sort(np.linalg.eigvals(0.5 * fd.diff_matrix(s, 2, 2, fd.NEUMANN_BC)).real)
    assert np.abs(got - want).max() <= 1e-9 * max(np.abs(want).max(), 1.0)
    assert np.allclose(fd.trapezoid_weights([0.0, 1.0, 3.0, 4.0]), [0.5, 1.5, 1.5, 0.5], atol=1e-15)
    with pytest.raises(InvalidGridError):
        fd.trapezoid_weights([0.0, 2.0, 1.0])


@pytest.mark.gpu
def test_operator_actions_on_device():
    assert np.abs(km.matvec(fd.heat_factors(4, 2), np.ones((4, 4, 4)))).max() <= 1e-13
    op = fd.pipeflow_factors(8)
    u = np.asfortranarray(np.random.default_rng(0).standard_normal((8, 8)))
    want = km.assemble_full(op) @ u.ravel(order="F")
    assert np.abs(km.matvec(op, u).ravel(order="F") - want).max() <= 1e-12 * np.abs(want).max()


# ------------------------------------------------------------------------ linalg (test_linalg.py)


def test_linalg_helpers():
    rng = np.random.default_rng(3)
    a, b = rng.standard_normal((4, 3)), rng.standard_normal((3, 5))
    assert np.allclose(km.matmul(a, b), a @ b)
    with pytest.raises(ShapeError):
        km.matmul(a, a)
    assert km.one_norm(np.array([[1.0, -2.0], [3.0, 4.0]])) == 6.0
    m = rng.standard_normal((5, 5)) + 5 * np.eye(5)
    rhs = rng.standard_normal(5)
    assert np.allclose(m @ km.solve(m, rhs), rhs)
    with pytest.raises(SingularMatrixError):
        km.solve(np.zeros((2, 2)), np.ones(2))
    with pytest.raises(ShapeError):
        km.solve(np.ones((2, 3)), np.ones(2))
    with pytest.raises(ShapeError):
        km.solve(np.eye(2), np.ones(3))
    assert np.array_equal(km.matexp(np.zeros((3, 3))), np.eye(3))
    assert km.matexp(np.eye(2)).dtype == np.float64
    with pytest.raises(InvalidInputError):
        km.matexp(np.array([[np.nan]]))
    with pytest.raises(ShapeError):
        km.matexp(np.ones((2, 3)))
