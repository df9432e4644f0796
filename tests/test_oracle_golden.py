"""CPU: pin the oracle (oracle/kronmode_oracle.py) and the package's host
builders against golden vectors produced by the reference itself
(tests/golden/make_golden.py).  No GPU, no /root/reference at run time."""

import math

import numpy as np
import pytest

from conftest import golden
from oracle import kronmode_oracle as orc


def _close(got, want, tol):
    want = np.asarray(want)
    scale = max(np.abs(want).max(), 1e-300)
    assert np.abs(np.asarray(got) - want).max() <= tol * scale


MUMODE_CASES = sorted({k.split("__")[0] for k in golden("mumode") if not k.startswith("tucker")})


@pytest.mark.parametrize("case", MUMODE_CASES)
def test_oracle_mu_mode_product_matches_reference(case):
    g = golden("mumode")
    got = orc.mu_mode_product(g[f"{case}__u"], g[f"{case}__mat"], int(g[f"{case}__mu"]))
    want = g[f"{case}__out"]
    assert got.dtype == want.dtype and got.shape == want.shape
    _close(got, want, 1e-15 if want.dtype in (np.float64, np.complex128) else 1e-6)


def test_oracle_tucker_skips_none():
    g = golden("mumode")
    got = orc.tucker(g["tucker_none__u"], [g["tucker_none__m0"], None, g["tucker_none__m2"]])
    _close(got, g["tucker_none__out"], 1e-15)


def test_oracle_step_and_ten_steps():
    g = golden("step")
    exps = [g[f"schrod16__e{i}"] for i in range(3)]
    _close(orc.step(exps, g["schrod16__u"]), g["schrod16__out"], 1e-15)
    v = g["schrod16__u"]
    for _ in range(10):
        v = orc.step(exps, v)
    _close(v, g["schrod16__out10"], 1e-14)
    _close(orc.step([g["heat16__e0"]] * 3, g["heat16__u"]), g["heat16__out"], 1e-15)


def test_oracle_hermite_transforms():
    g = golden("hermite")
    phi, w = g["herm12__phi"], g["herm12__w"]
    fwd = orc.forward_transform([phi] * 3, [w] * 3, g["herm12__values"])
    _close(fwd, g["herm12__forward"], 1e-14)
    _close(orc.inverse_transform([phi.T] * 3, g["herm12__forward"]), g["herm12__inverse"], 1e-14)


def test_oracle_gpe_strang_matches_reference():
    g = golden("gpe")
    exps = [g[f"gpe16__e{i}"] for i in range(3)]
    ws = [g[f"gpe16__w{i}"] for i in range(3)]
    p = orc.gpe_strang_step(exps, ws, g["gpe16__psi0"], 0.1)
    _close(p, g["gpe16__out1"], 1e-15)
    for _ in range(4):
        p = orc.gpe_strang_step(exps, ws, p, 0.1)
    _close(p, g["gpe16__out5"], 1e-14)
    p64 = orc.gpe_strang_step([e.astype(np.complex64) for e in exps], ws,
                              g["gpe16__psi0"].astype(np.complex64), 0.1)
    assert p64.dtype == g["gpe16c64__out1"].dtype == np.complex128
    _close(p64, g["gpe16c64__out1"], 1e-7)


def test_oracle_rel_l2():
    a = np.ones((3, 4))
    assert orc.rel_l2(a, a) == 0.0
    assert math.isclose(orc.rel_l2(2 * a, a), 1.0)


# ---- the package's host builders (inputs of the hot path) vs the reference

def test_host_heat_factors_match_reference():
    from paper_2103_01691_b200 import fd

    g = golden("builders")
    for p in (2, 4):
        _close(fd.heat_factors(16, p).factors[0], g[f"heat_d2_n16_p{p}"], 1e-14)
    _close(fd.heat_factors(16, np.inf).factors[0], g["heat_d2_n16_pinf"], 1e-14)
    st = golden("step")
    assert np.array_equal(fd.heat_factors(16, 2).factors[0], st["schrod16__d2"])


def test_host_pipeflow_factors_match_reference():
    from paper_2103_01691_b200 import fd

    g = golden("builders")
    a0, a1 = fd.pipeflow_factors(16).factors
    _close(a0, g["pipe16__a0"], 1e-13)
    _close(a1, g["pipe16__a1"], 1e-13)


def test_host_hermite_basis_matches_reference():
    from paper_2103_01691_b200 import hermite

    g = golden("hermite")
    for k in (16, 64):
        b = hermite.hermite_basis(k)
        assert np.array_equal(b.nodes, g[f"basis{k}__nodes"])
        assert np.array_equal(b.mod_weights, g[f"basis{k}__w"])
        assert np.array_equal(b.phi, g[f"basis{k}__phi"])


def test_host_gpe_setup_matches_reference():
    from paper_2103_01691_b200 import problems

    g = golden("gpe")
    grids, lin_op, weights = problems.gpe_setup(16)
    for i in range(3):
        assert np.array_equal(grids[i].points, g[f"gpe16__x{i}"])
        assert np.array_equal(weights[i], g[f"gpe16__w{i}"])
        _close(lin_op.factors[i], g[f"gpe16__a{i}"], 1e-14)
    psi = problems.weighted_vortex_state(grids, weights)
    _close(psi, g["gpe16__psi0"], 1e-15)


def test_host_prepare_matches_reference():
    from paper_2103_01691_b200 import kron

    g = golden("step")
    cache = kron.prepare(kron.KroneckerOp((1j * g["schrod16__d2"],) * 3), 0.01)
    for i in range(3):
        assert np.array_equal(cache.exps[i], g[f"schrod16__e{i}"])


def test_heat_closed_form_kat():
    # test_problems.py:61-67 closed form; BASELINE.md KAT values
    def err(n):
        h = 2 * np.pi / n
        lam = (2 * np.cos(h) - 2) / h**2
        return abs(np.exp(lam) - np.exp(-1.0)) / np.exp(-1.0)

    assert math.isclose(err(16), float(golden("step")["heat16__error"]), rel_tol=1e-9)
    for n, want in [(200, 8.225e-5), (300, 3.655e-5), (400, 2.056e-5), (500, 1.316e-5)]:
        assert abs(err(n) - want) <= 1e-3 * want
