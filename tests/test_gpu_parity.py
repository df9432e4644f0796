"""GPU parity: the CUDA path (through the C ABI) against the reference's golden
vectors and the CPU oracle on the same seeded inputs.

Bars (north star): relative l2 <= 1e-12 for complex128/float64 and <= 1e-5
for complex64/float32; bitwise where the reference's own tests are bitwise
(identity, tau = 0).  Full-size (256^3) cases are checked against the oracle
directly and through size-independent properties (unitarity, plane-wave
eigenvectors, direction-order invariance).
"""

import numpy as np
import pytest

import paper_2103_01691_b200 as km
from conftest import golden
from oracle import kronmode_oracle as orc

pytestmark = pytest.mark.gpu

TOL = {np.dtype(np.complex128): 1e-12, np.dtype(np.float64): 1e-12,
       np.dtype(np.complex64): 1e-5, np.dtype(np.float32): 1e-5}


def rel(a, b):
    return orc.rel_l2(a, b)


def crand(rng, shape, dtype=np.complex128):
    return np.asfortranarray((rng.standard_normal(shape) + 1j * rng.standard_normal(shape)).astype(dtype))


def schrod_cache(n, tau=0.01):
    d2 = km.heat_factors(n, 2).factors[0]
    return km.prepare(km.KroneckerOp((1j * d2,) * 3), tau)


# ------------------------------------------------------------ golden vectors

MUMODE_CASES = sorted({k.split("__")[0] for k in golden("mumode") if not k.startswith("tucker")})


@pytest.mark.parametrize("case", MUMODE_CASES)
def test_mu_mode_product_matches_reference_golden(case):
    g = golden("mumode")
    want = g[f"{case}__out"]
    got = km.mu_mode_product(g[f"{case}__u"], g[f"{case}__mat"], int(g[f"{case}__mu"]))
    assert got.dtype == want.dtype and got.shape == want.shape
    assert got.flags.f_contiguous
    assert rel(got, want) <= TOL[want.dtype]


def test_tucker_none_slot_golden():
    g = golden("mumode")
    got = km.tucker(g["tucker_none__u"], [g["tucker_none__m0"], None, g["tucker_none__m2"]])
    assert rel(got, g["tucker_none__out"]) <= 1e-12


def test_step_golden_one_and_ten_steps():
    g = golden("step")
    cache = km.PropagatorCache(0.01, tuple(g[f"schrod16__e{i}"] for i in range(3)))
    assert rel(km.step(cache, g["schrod16__u"]), g["schrod16__out"]) <= 1e-12
    v = g["schrod16__u"]
    for _ in range(10):
        v = km.step(cache, v)
    assert rel(v, g["schrod16__out10"]) <= 1e-12
    heat = km.PropagatorCache(0.1, (g["heat16__e0"],) * 3)
    assert rel(km.step(heat, g["heat16__u"]), g["heat16__out"]) <= 1e-12


def test_hermite_transforms_golden():
    g = golden("hermite")
    b = km.hermite_basis(12)
    bases = (b,) * 3
    fwd = km.forward_transform(bases, g["herm12__values"])
    assert fwd.dtype == g["herm12__forward"].dtype
    assert rel(fwd, g["herm12__forward"]) <= 1e-12
    assert rel(km.inverse_transform(bases, g["herm12__forward"]), g["herm12__inverse"]) <= 1e-12
    pts = [g["herm12__pts0"], g["herm12__pts1"], g["herm12__pts2"]]
    got = km.inverse_transform(bases, g["herm12__forward"], eval_points=pts)
    assert got.shape == (7, 5, 2)
    assert rel(got, g["herm12__inverse_pts"]) <= 1e-12


def test_hkp_pipeline_golden():
    g = golden("hermite")
    kb = km.hermite_basis(10)
    c0 = km.forward_transform((kb,) * 3, g["hkp10__psi0"])
    assert rel(c0, g["hkp10__c0"]) <= 1e-12
    cache = km.PropagatorCache(1.0, tuple(g[f"hkp10__e{i}"] for i in range(3)))
    ct = km.step(cache, c0)
    assert rel(ct, g["hkp10__ct"]) <= 1e-12
    assert rel(km.inverse_transform((kb,) * 3, ct), g["hkp10__values"]) <= 1e-12


def test_magnus_golden():
    from paper_2103_01691_b200.problems import hkmp_factors

    g = golden("hermite")
    basis = km.hermite_basis(8)
    u = g["hkmp8__c0"]
    tau = 0.5 / 4
    for s in range(4):
        u = km.magnus_midpoint_step(lambda t: hkmp_factors(basis, t), u, s * tau, tau)
    assert rel(u, g["hkmp8__out"]) <= 1e-12


def test_gpe_strang_golden():
    g = golden("gpe")
    cache = km.PropagatorCache(0.1, tuple(g[f"gpe16__e{i}"] for i in range(3)))
    ws = [g[f"gpe16__w{i}"] for i in range(3)]
    p = km.gpe_strang_step(cache, ws, g["gpe16__psi0"], 0.1)
    assert p.dtype == np.complex128
    assert rel(p, g["gpe16__out1"]) <= 1e-12
    for _ in range(4):
        p = km.gpe_strang_step(cache, ws, p, 0.1)
    assert rel(p, g["gpe16__out5"]) <= 1e-12
    c64 = km.PropagatorCache(0.1, tuple(e.astype(np.complex64) for e in cache.exps))
    p64 = km.gpe_strang_step(c64, ws, g["gpe16__psi0"].astype(np.complex64), 0.1)
    assert p64.dtype == g["gpe16c64__out1"].dtype == np.complex128
    # the reference promotes the state to complex128 in the opening phase (with a float32
    # density, problems.py:543-545), so the complex128 bar applies
    assert rel(p64, g["gpe16c64__out1"]) <= 1e-12


# ------------------------------------------------ reference test semantics

def test_identity_is_bitwise_identity():
    rng = np.random.default_rng(7)
    for u in (np.asfortranarray(rng.random((3, 4, 2)) + 0.5), crand(rng, (3, 4, 2))):
        for mu in (1, 2, 3):
            got = km.mu_mode_product(u, np.eye(u.shape[mu - 1]), mu)
            assert np.array_equal(got, u)


def test_row_permutation_exact():
    u = np.array([[1.0, 2.0], [3.0, 4.0]])
    swap = np.array([[0.0, 1.0], [1.0, 0.0]])
    assert np.array_equal(km.mu_mode_product(u, swap, 1), np.array([[3.0, 4.0], [1.0, 2.0]]))


def test_random_small_shapes_vs_oracle():
    rng = np.random.default_rng(123)
    for trial in range(60):
        d = int(rng.integers(1, 5))
        shape = tuple(int(x) for x in rng.integers(1, 5, size=d))
        mu = int(rng.integers(1, d + 1))
        rows = int(rng.integers(1, 5))
        u = rng.standard_normal(shape)
        if trial % 2:
            u = u + 1j * rng.standard_normal(shape)
        mat = rng.standard_normal((rows, shape[mu - 1]))
        got = km.mu_mode_product(u, mat, mu)
        want = orc.mu_mode_product(u, mat, mu)
        scale = max(np.abs(want).max(), 1.0)
        assert np.abs(got - want).max() <= 1e-14 * scale


def test_single_precision_preserved():
    rng = np.random.default_rng(5)
    u = rng.standard_normal((4, 4)).astype(np.float32)
    mat = rng.standard_normal((4, 4)).astype(np.float32)
    got = km.mu_mode_product(u, mat, 1)
    assert got.dtype == np.float32
    assert rel(got, orc.mu_mode_product(u, mat, 1)) <= 1e-5


def test_complex_promotion():
    rng = np.random.default_rng(3)
    u = rng.standard_normal((2, 3))
    mat = rng.standard_normal((3, 3)) + 1j * rng.standard_normal((3, 3))
    got = km.mu_mode_product(u, mat, 2)
    assert got.dtype == np.complex128
    assert np.abs(got - orc.mu_mode_product(u, mat, 2)).max() <= 1e-14


def test_flop_counter_exact():
    rng = np.random.default_rng(12)
    dims = (3, 4, 5)
    op = km.KroneckerOp(tuple(rng.standard_normal((m, m)) for m in dims))
    cache = km.prepare(op, 0.2)
    with km.count_flops() as fc:
        km.step(cache, np.asfortranarray(rng.standard_normal(dims)))
    assert fc.macs == sum(60 * m for m in dims)


def test_step_zero_increment_bitwise():
    rng = np.random.default_rng(6)
    op = km.KroneckerOp((rng.standard_normal((3, 3)), rng.standard_normal((4, 4))))
    u = np.asfortranarray(rng.standard_normal((3, 4)))
    assert np.array_equal(km.step(km.prepare(op, 0.0), u), u)


def test_step_matches_dense_exponential():
    rng = np.random.default_rng(9)
    for trial in range(8):
        dims = tuple(int(rng.integers(2, 5)) for _ in range(int(rng.integers(2, 4))))
        facs = []
        for m in dims:
            a = rng.standard_normal((m, m))
            if trial % 2:
                a = a + 1j * rng.standard_normal((m, m))
            facs.append(a)
        op = km.KroneckerOp(tuple(facs))
        u = np.asfortranarray(rng.standard_normal(dims))
        tau = float(rng.uniform(0.1, 1.0))
        got = km.step(km.prepare(op, tau), u).ravel(order="F")
        want = km.matexp(tau * km.assemble_full(op)) @ u.ravel(order="F")
        assert np.linalg.norm(got - want) <= 1e-12 * np.linalg.norm(want)


def test_matvec_vs_dense():
    rng = np.random.default_rng(3)
    op = km.KroneckerOp(tuple(rng.standard_normal((m, m)) + 1j * rng.standard_normal((m, m))
                              for m in (3, 2, 4)))
    u = np.asfortranarray(rng.standard_normal((3, 2, 4)))
    want = km.assemble_full(op) @ u.ravel(order="F")
    got = km.matvec(op, u).ravel(order="F")
    assert np.abs(got - want).max() <= 1e-13 * np.abs(want).max()


def test_norms_on_device():
    rng = np.random.default_rng(12)
    u = rng.standard_normal((3, 4)) + 1j * rng.standard_normal((3, 4))
    w1, w2 = rng.random(3) + 0.1, rng.random(4) + 0.1
    want = np.sqrt(sum(w1[i] * w2[j] * abs(u[i, j]) ** 2 for i in range(3) for j in range(4)))
    assert km.norm(u, "weighted_two", weights=[w1, w2]) == pytest.approx(want, rel=1e-13)
    assert km.norm(u, "two") == pytest.approx(np.linalg.norm(u), rel=1e-14)
    assert km.norm(u, "max") == pytest.approx(np.abs(u).max(), rel=1e-15)


def test_gpe_tau_zero_identity_bitwise_and_modulus():
    rng = np.random.default_rng(2)
    _, lin_op, weights = km.gpe_setup(16)
    psi = crand(rng, (16, 16, 16))
    got = km.gpe_strang_step(km.prepare(lin_op, 0.0), weights, psi, 0.0)
    assert np.array_equal(got, psi)
    stepped = km.gpe_strang_step(km.prepare(lin_op, 0.0), weights, psi, 0.3)
    assert np.abs(np.abs(stepped) - np.abs(psi)).max() <= 1e-14


def test_gpe_unit_background_stationary():
    n = 32
    _, lin_op, weights = km.gpe_setup(n)
    psi = np.ones((n, n, n), dtype=complex, order="F")
    for ax, w in enumerate(weights):
        psi = psi * np.sqrt(w).reshape((1,) * ax + (n,) + (1,) * (2 - ax))
    start = np.asfortranarray(psi)
    cache = km.prepare(lin_op, 0.1)
    p = start
    for _ in range(10):
        p = km.gpe_strang_step(cache, weights, p, 0.1)
    assert np.abs(p - start).max() <= 1e-12 * np.abs(start).max()


# ------------------------------------------------ config-scale parity

def test_config1_schrodinger_64_ten_steps_vs_oracle():
    n = 64
    rng = np.random.default_rng(0)
    u = crand(rng, (n,) * 3)
    cache = schrod_cache(n)
    got, want = u, u
    for _ in range(10):
        got = km.step(cache, got)
        want = orc.step(cache.exps, want)
    assert rel(got, want) <= 1e-12


def test_config2_pipeflow_1024_vs_oracle():
    n = 1024
    op = km.pipeflow_factors(n)
    cache = km.prepare(op, 4.0 / 8)
    rho, z = np.linspace(0.1, 5.0, n), np.linspace(0.0, 8.0, n)
    c0 = np.asfortranarray(np.exp(-8.0 * (rho - 2.55) ** 2)[:, None] * np.exp(-8.0 * (z - 1.5) ** 2)[None, :])
    got = km.step(cache, c0)
    assert got.dtype == np.float64
    assert rel(got, orc.step(cache.exps, c0)) <= 1e-12
    c0c = np.asfortranarray(c0 * (1 + 1j))
    assert rel(km.step(cache, c0c), orc.step(cache.exps, c0c)) <= 1e-12


def test_complex64_step_vs_oracle():
    n = 64
    rng = np.random.default_rng(1)
    u = crand(rng, (n,) * 3, np.complex64)
    cache = schrod_cache(n)
    c64 = km.PropagatorCache(0.01, tuple(e.astype(np.complex64) for e in cache.exps))
    got = km.step(c64, u)
    assert got.dtype == np.complex64
    assert rel(got, orc.step(c64.exps, u)) <= 1e-5


@pytest.mark.slow
def test_headline_256_step_vs_oracle_and_properties():
    n = 256
    rng = np.random.default_rng(0)
    u = crand(rng, (n,) * 3)
    cache = schrod_cache(n)
    got = km.step(cache, u)
    assert rel(got, orc.step(cache.exps, u)) <= 1e-12
    # E_mu is unitary (exp of i * symmetric): the step preserves the 2-norm
    assert abs(np.linalg.norm(got.ravel()) / np.linalg.norm(u.ravel()) - 1) <= 1e-12
    # direction order is immaterial (kron.py:115-116)
    rev = u
    for mu in (3, 2, 1):
        rev = km.mu_mode_product(rev, cache.exps[mu - 1], mu)
    assert rel(rev, got) <= 1e-12


@pytest.mark.slow
def test_headline_256_plane_wave_eigenvector():
    n, steps, tau = 256, 3, 0.01
    h = 2 * np.pi / n
    x = h * np.arange(n)
    ks = (1, 2, 3)
    u = np.exp(1j * ks[0] * x)[:, None, None] * np.exp(1j * ks[1] * x)[None, :, None] \
        * np.exp(1j * ks[2] * x)[None, None, :]
    u = np.asfortranarray(u)
    lam = sum((2 * np.cos(k * h) - 2) / h**2 for k in ks)
    cache = schrod_cache(n, tau)
    v = u
    for _ in range(steps):
        v = km.step(cache, v)
    assert rel(v, np.exp(1j * tau * steps * lam) * u) <= 1e-12


def test_tdpot_strang_vs_oracle():
    from paper_2103_01691_b200.hermite import physical_propagator
    from paper_2103_01691_b200.problems import schrodinger_initial_state

    k = 32
    b = km.hermite_basis(k)
    tau = 0.02
    p = physical_propagator(b, tau)
    cache = km.PropagatorCache(tau, (p, p, p))
    psi = schrodinger_initial_state((b.nodes,) * 3)
    got, want = psi, psi
    for s in range(3):
        got = km.tdpot_strang_step(cache, b.nodes, got, s * tau, tau)
        want = orc.tdpot_strang_step(cache.exps, b.nodes, want, s * tau, tau)
    assert rel(got, want) <= 1e-12


@pytest.mark.parametrize("n,direction", [(32, 3), (256, 3), (48, 2), (40, 1)])
def test_direction_diagonal_phase_ops(n, direction):
    """KM_OP_DIAG as the pre pass and as the fused epilogue of the last product (the C-ABI op
    behind direction-diagonal phases): psi -> f_b[i_dir] * (E-step(f_a[i_dir] * psi))."""
    from paper_2103_01691_b200 import _device as dv
    from paper_2103_01691_b200.problems import _diag_op
    from paper_2103_01691_b200.tensor import run_tucker

    rng = np.random.default_rng(n + direction)
    shape = (n,) * 3
    u = np.asfortranarray(rng.standard_normal(shape) + 1j * rng.standard_normal(shape))
    mats = [(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / np.sqrt(n) for _ in range(3)]
    f_a = np.exp(1j * rng.standard_normal(n))
    f_b = np.exp(1j * rng.standard_normal(n))
    import torch

    dev = torch.device("cuda", 0)
    fa_d, fb_d = (dv.cached_vector(f, np.complex128, dev) for f in (f_a, f_b))
    got = run_tucker(u, mats, pre=_diag_op(shape, fa_d, direction - 1), post=_diag_op(shape, fb_d, direction - 1),
                     keepalive=(fa_d, fb_d))
    bshape = [1, 1, 1]
    bshape[direction - 1] = n
    want = orc.step(mats, u * f_a.reshape(bshape)) * f_b.reshape(bshape)
    assert rel(got, want) <= 1e-12


@pytest.mark.parametrize("m,k,same", [(24, 40, False), (64, 64, True)])
def test_diag_phase_fold_matches_numpy(m, k, same):
    """km_diag_phase_fold (config 4's flows folded into a factor) against the host formula
    (f_b[i] * E[i, j]) * f_a[j] with f = exp(-1j * x * c)."""
    import ctypes

    import torch

    from paper_2103_01691_b200 import _device as dv, _native

    rng = np.random.default_rng(m + k)
    E = rng.standard_normal((m, k)) + 1j * rng.standard_normal((m, k))
    xr = rng.standard_normal(m) * 3
    xc = xr if same else rng.standard_normal(k) * 3
    c_a, c_b = 0.0123, 0.0456
    dev_ = torch.device("cuda", 0)
    e_d = torch.from_numpy(E).to(dev_)
    out = torch.empty_like(e_d)
    xr_d, xc_d = torch.from_numpy(xr).to(dev_), torch.from_numpy(xc).to(dev_)
    _native.check(_native.lib().km_diag_phase_fold(e_d.data_ptr(), out.data_ptr(), m, k, xr_d.data_ptr(),
                                                   xc_d.data_ptr(), c_a, c_b,
                                                   ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
    want = (np.exp(-1j * xr * c_b)[:, None] * E) * np.exp(-1j * xc * c_a)[None, :]
    assert rel(out.cpu().numpy(), want) <= 1e-15
    with pytest.raises(Exception):
        _native.check(_native.lib().km_diag_phase_fold(e_d.data_ptr(), e_d.data_ptr(), m, k, xr_d.data_ptr(),
                                                       xc_d.data_ptr(), c_a, c_b, None))


def test_physical_propagator_equals_transform_step_transform():
    from paper_2103_01691_b200.hermite import physical_propagator

    k = 16
    b = km.hermite_basis(k)
    rng = np.random.default_rng(4)
    vals = crand(rng, (k,) * 3)
    tau = 0.3
    harm = km.KroneckerOp((-1j * np.diag(np.arange(k) + 0.5),) * 3)
    via = km.inverse_transform((b,) * 3, km.step(km.prepare(harm, tau), km.forward_transform((b,) * 3, vals)))
    p = physical_propagator(b, tau)
    direct = km.step(km.PropagatorCache(tau, (p,) * 3), vals)
    assert rel(direct, via) <= 1e-12


# ------------------------------------------------ device tensors in / out

def test_torch_tensors_stay_on_device():
    import torch

    from paper_2103_01691_b200 import _device as dv

    n = 32
    rng = np.random.default_rng(8)
    u = crand(rng, (n,) * 3)
    cache = schrod_cache(n)
    t = dv.to_device(u, np.complex128, torch.device("cuda"))
    assert dv.is_fortran(t)
    out = km.step(cache, t)
    assert isinstance(out, torch.Tensor) and out.is_cuda and dv.is_fortran(out)
    assert rel(dv.to_host(out), orc.step(cache.exps, u)) <= 1e-12


def test_gpe_strang_run_equals_step_loop():
    g = golden("gpe")
    cache = km.PropagatorCache(0.1, tuple(g[f"gpe16__e{i}"] for i in range(3)))
    ws = [g[f"gpe16__w{i}"] for i in range(3)]
    run = km.gpe_strang_run(cache, ws, g["gpe16__psi0"], 0.1, 5)
    assert rel(run, g["gpe16__out5"]) <= 1e-12
    p = g["gpe16__psi0"]
    for _ in range(5):
        p = km.gpe_strang_step(cache, ws, p, 0.1)
    assert np.array_equal(run, p)


def test_gpe_strang_run_256_vs_step_loop():
    import torch

    from paper_2103_01691_b200 import _device as dv
    from paper_2103_01691_b200.problems import weighted_vortex_state

    n = 256
    grids, lin_op, weights = km.gpe_setup(n)
    psi = weighted_vortex_state(grids, weights)
    cache = km.prepare(lin_op, 0.1)
    t = dv.to_device(psi, np.complex128, torch.device("cuda", 0))
    run = dv.to_host(km.gpe_strang_run(cache, weights, t, 0.1, 3))
    p = t
    for _ in range(3):
        p = km.gpe_strang_step(cache, weights, p, 0.1)
    assert np.array_equal(run, dv.to_host(p))


# ------------------------------------------------ device norms (km_norm)

def test_relative_error_reference_semantics():
    # test_problems.py:31-47
    a = np.array([1.0, 2.0, 3.0])
    assert km.relative_error(a, a) == 0.0
    assert km.relative_error(2 * a, a, "two") == pytest.approx(1.0, rel=1e-15)
    with pytest.raises(km.InvalidReferenceError):
        km.relative_error(a, np.zeros(3))
    with pytest.raises(km.ShapeError):
        km.relative_error(a, np.ones(4))


@pytest.mark.parametrize("kind", ["max", "two", "weighted_two"])
def test_norms_large_vs_numpy(kind):
    rng = np.random.default_rng(11)
    shape = (96, 80, 70)
    u = np.asfortranarray(rng.standard_normal(shape) + 1j * rng.standard_normal(shape))
    ref = np.asfortranarray(u + 1e-3 * rng.standard_normal(shape))
    ws = [rng.random(n) + 0.1 for n in shape]
    if kind == "max":
        want_n, want_e = np.abs(u).max(), np.abs(u - ref).max() / np.abs(ref).max()
    elif kind == "two":
        want_n, want_e = np.linalg.norm(u.ravel()), np.linalg.norm((u - ref).ravel()) / np.linalg.norm(ref.ravel())
    else:
        wp = orc.weight_product(ws, shape)
        want_n = np.sqrt(np.sum(wp * np.abs(u) ** 2))
        want_e = np.sqrt(np.sum(wp * np.abs(u - ref) ** 2)) / np.sqrt(np.sum(wp * np.abs(ref) ** 2))
    w = ws if kind == "weighted_two" else None
    assert km.norm(u, kind, w) == pytest.approx(want_n, rel=1e-13)
    assert km.relative_error(u, ref, kind, w) == pytest.approx(want_e, rel=1e-12)


@pytest.mark.parametrize("dtype,tol", [(np.complex128, 0.0), (np.float64, 0.0), (np.complex64, 1e-5)])
def test_matvec_accumulates_like_the_reference(dtype, tol):
    """kron.matvec accumulates the d products in the epilogues (km_mumode_split accumulate):
    the same ``out += p`` roundings as kron.py:99-101 (bitwise in double precision against
    the oracle's products summed the reference's way), 3 launches, no temporaries."""
    rng = np.random.default_rng(21)
    shape = (48, 40, 36)
    cplx = np.dtype(dtype).kind == "c"
    u = crand(rng, shape, dtype) if cplx else np.asfortranarray(rng.standard_normal(shape).astype(dtype))
    facs = [rng.standard_normal((n, n)).astype(dtype) + (1j * rng.standard_normal((n, n)) if cplx else 0)
            for n in shape]
    facs = [f.astype(dtype) for f in facs]
    op = km.KroneckerOp(tuple(facs))
    got = km.matvec(op, u)
    want = km.mu_mode_product(u, facs[0], 1)
    for mu in (2, 3):
        want = want + km.mu_mode_product(u, facs[mu - 1], mu)
    assert got.dtype == want.dtype
    if tol == 0.0:
        assert np.array_equal(got, want)
    ref = orc.mu_mode_product(u, facs[0], 1)
    for mu in (2, 3):
        ref += orc.mu_mode_product(u, facs[mu - 1], mu)
    assert rel(got, ref) <= (1e-12 if tol == 0.0 else tol)


@pytest.mark.parametrize("shape,dtype", [((33, 17, 5), np.complex128), ((7, 40, 9), np.float64),
                                         ((19, 3, 31), np.complex64), ((65, 1, 2), np.complex128),
                                         ((256, 256, 256), np.complex128)])
def test_matvec_ragged_and_full_size(shape, dtype):
    """The accumulating epilogue on ragged tiles (edge rows / fibers), a size-1 direction, and
    the 256^3 TMA kernel, against the reference's out += p (kron.py:94-102) on the oracle."""
    rng = np.random.default_rng(sum(shape))
    cplx = np.dtype(dtype).kind == "c"
    u = crand(rng, shape, dtype) if cplx else np.asfortranarray(rng.standard_normal(shape).astype(dtype))
    facs = tuple(((rng.standard_normal((n, n)) + (1j * rng.standard_normal((n, n)) if cplx else 0)) / np.sqrt(n))
                 .astype(dtype) for n in shape)
    got = km.matvec(km.KroneckerOp(facs), u)
    want = orc.mu_mode_product(u, facs[0], 1)
    for mu in range(2, 4):
        want = want + orc.mu_mode_product(u, facs[mu - 1], mu)
    assert got.dtype == want.dtype and got.shape == want.shape
    assert rel(got, want) <= TOL[np.dtype(dtype)]
