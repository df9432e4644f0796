"""GPU matrix exponential (expm.py) against scipy's, and the
Magnus midpoint scheme with device exponentials against the reference's golden run."""

import numpy as np
import pytest
import scipy.linalg

import paper_2103_01691_b200 as km
from conftest import golden
from oracle import kronmode_oracle as orc
from paper_2103_01691_b200 import _device as dv
from paper_2103_01691_b200.expm import matexp_device, prepare_device
from paper_2103_01691_b200.problems import hkmp_factors

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,scale,cplx", [(1, 0.3, False), (8, 0.1, False), (33, 2.0, True), (128, 10.0, True),
                                          (256, 40.0, True), (200, 0.0, True)])
def test_matexp_device_vs_scipy(n, scale, cplx):
    rng = np.random.default_rng(n)
    a = rng.standard_normal((n, n))
    if cplx:
        a = a + 1j * rng.standard_normal((n, n))
    a *= scale / max(np.linalg.norm(a, 1), 1e-300)
    got = dv.to_host(matexp_device(a))
    want = scipy.linalg.expm(a)
    assert np.linalg.norm(got - want) <= 1e-13 * np.linalg.norm(want)


def test_skew_hermitian_generator_unitary():
    b = km.hermite_basis(64)
    a = -1j * 0.05 * (np.diag(np.arange(64) + 0.5) + 0.7 * km.position_operator(b))
    e = dv.to_host(matexp_device(a))
    assert np.abs(e.conj().T @ e - np.eye(64)).max() <= 1e-13


def test_magnus_with_device_expm_matches_reference_golden():
    g = golden("hermite")
    basis = km.hermite_basis(8)
    u = g["hkmp8__c0"]
    tau = 0.5 / 4
    for s in range(4):
        u = km.magnus_midpoint_step(lambda t: hkmp_factors(basis, t), u, s * tau, tau, device_expm=True)
    assert orc.rel_l2(u, g["hkmp8__out"]) <= 1e-12


def test_device_cache_step_matches_host_cache():
    n = 64
    d2 = km.heat_factors(n, 2).factors[0]
    op = km.KroneckerOp((1j * d2,) * 3)
    rng = np.random.default_rng(1)
    u = np.asfortranarray(rng.standard_normal((n,) * 3) + 1j * rng.standard_normal((n,) * 3))
    host = km.step(km.prepare(op, 0.01), u)
    dev = km.step(prepare_device(op, 0.01), u)
    assert orc.rel_l2(dev, host) <= 1e-13
    assert prepare_device(op, 0.01).exps[0].shape == (n, n)


def test_device_cache_step_with_device_tensor():
    """A device-resident state through a DevicePropagatorCache takes kron.step's prebuilt-call
    path (the cache's memo of StepPlans), as the Magnus driver does with device tensors."""
    n = 64
    d2 = km.heat_factors(n, 2).factors[0]
    op = km.KroneckerOp((1j * d2,) * 3)
    rng = np.random.default_rng(2)
    u = np.asfortranarray(rng.standard_normal((n,) * 3) + 1j * rng.standard_normal((n,) * 3))
    cache = prepare_device(op, 0.01)
    t = dv.to_device(u, np.complex128, dv.device())
    for _ in range(2):  # the second call reuses the memoised plan
        got = km.step(cache, t)
    want = orc.step(km.prepare(op, 0.01).exps, u)
    assert orc.rel_l2(dv.to_host(got), want) <= 1e-13
    basis = km.hermite_basis(8)
    c0 = dv.to_device(np.asfortranarray(golden("hermite")["hkmp8__c0"]), np.complex128, dv.device())
    c = km.magnus_midpoint_step(lambda s: hkmp_factors(basis, s), c0, 0.0, 0.125, device_expm=True)
    ref = km.magnus_midpoint_step(lambda s: hkmp_factors(basis, s), golden("hermite")["hkmp8__c0"], 0.0, 0.125)
    assert orc.rel_l2(dv.to_host(c), ref) <= 1e-12
